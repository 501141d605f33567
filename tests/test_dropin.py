"""Drop-in boundary: the reference's unmodified experiments.hpp / tuner.hpp / synth.hpp
compiled against include/aiwc/forest.hpp (this repo), linked to libaiwc_cuda.so
(oracle/_ref/dropin_test, built by `make -C oracle dropin` where /root/reference exists)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")
# canonical model JSON of the C1 500/6/5 forest: 17,820,410 bytes, FNV-1a64 below
# (SURVEY.md section 8c golden, reproduced by oracle/_ref in tests/golden)
C1_JSON_FNV = 0x22EFBC8C4B207134
C1_JSON_SIZE = 17820410

needs_bin = pytest.mark.skipif(not os.path.exists(BIN), reason="dropin_test not built")


@needs_bin
def test_dropin_binary_links_product_library():
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    line = [x for x in out.splitlines() if "libaiwc_cuda.so" in x]
    assert line and "not found" not in line[0]


@needs_bin
@pytest.mark.gpu
def test_reference_callers_run_unchanged_on_gpu(golden):
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    got = json.loads(r.stdout.strip().splitlines()[-1])
    assert got["json_fnv"] == C1_JSON_FNV and got["json_size"] == C1_JSON_SIZE
    c1 = golden["c1_500_6_5"]["oob"]
    assert got["oob_error_pct"] == c1[3] and got["r2"] == c1[4]
    assert got["oob_recomputed"] == c1[3]
    assert got["obj_505_30_9"] == golden["c1_505_30_9"]["oob"][3]
    c3 = golden["c3_50_6_5"]
    # the golden MAPE is numpy's (pairwise) mean, the binary sums in row order; the
    # per-row predictions themselves are compared bit-exactly in test_gpu_parity.py
    assert got["c3_50_mape"] == pytest.approx(c3["mape"], rel=1e-13)
    assert (got["pairs"], got["pairs_correct"]) == (c3["pairs"], c3["pairs_correct"])
    assert got["roundtrip"] is True


@needs_bin
@pytest.mark.gpu
def test_heatmap_scan_batches_concurrent_fits():
    """The reference's heatmap_scan (experiments.hpp:79-123), 12 SA chains on 12 threads,
    every objective a drop-in fit on ONE PreparedDataset: the library merges the chains'
    concurrent fits into one multi-forest launch per round.  The cells equal the
    reference's own run (tests/golden/heatmap_c1.json) bit for bit, and batching beats
    the same scan with every fit run alone (AIWC_FIT_BATCH=0)."""
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "heatmap_c1.json")))
    runs = {}
    for mode, env in (("serial", {"AIWC_FIT_BATCH": "0"}), ("batched", {})):
        r = subprocess.run([BIN, "heatmap"], capture_output=True, text=True, timeout=900,
                           env={**os.environ, **env})
        assert r.returncode == 0, r.stderr
        runs[mode] = json.loads(r.stdout.strip().splitlines()[-1])
        assert runs[mode]["evaluations"] == gold["evaluations"]
        assert runs[mode]["cells"] == gold["cells"], mode
    speedup = runs["serial"]["seconds"] / runs["batched"]["seconds"]
    print(f"heatmap_scan: serial {runs['serial']['seconds']:.3f} s, batched "
          f"{runs['batched']['seconds']:.3f} s, x{speedup:.2f}")
    assert speedup > 1.5  # measured 1.9-3.4x on B200 boxes (profiles/r2_heatmap_batching.txt)
