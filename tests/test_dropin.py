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
    secs = {"serial": [], "batched": []}
    # the batched scan's time depends on how the 12 threads' fits meet (0.9-2.5 s measured
    # on one box), so each mode runs twice and the best run is compared
    for mode, env in (("serial", {"AIWC_FIT_BATCH": "0"}), ("batched", {})) * 2:
        r = subprocess.run([BIN, "heatmap"], capture_output=True, text=True, timeout=900,
                           env={**os.environ, **env})
        assert r.returncode == 0, r.stderr
        run = json.loads(r.stdout.strip().splitlines()[-1])
        assert run["evaluations"] == gold["evaluations"]
        assert run["cells"] == gold["cells"], mode
        secs[mode].append(run["seconds"])
    speedup = min(secs["serial"]) / min(secs["batched"])
    print(f"heatmap_scan: serial {secs['serial']} s, batched {secs['batched']} s, "
          f"x{speedup:.2f}")
    assert speedup > 1.2  # measured 1.4-3.4x (profiles/r2_heatmap_batching.txt)


@needs_bin
@pytest.mark.gpu
def test_model_file_fast_path_is_byte_identical():
    """Forest::save / load write and read the canonical model bytes directly (no JSON DOM):
    byte-identical to the reference's to_json().dump() (the C1 500/6/5 model, FNV-1a
    pinned), and the loaded forest re-serialises to the same bytes."""
    r = subprocess.run([BIN, "json"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    got = json.loads(r.stdout.strip().splitlines()[-1])
    assert got["identical"] is True
    assert got["bytes"] == C1_JSON_SIZE and got["fnv"] == C1_JSON_FNV
    print(f"model file: DOM write {got['dom_write_ms']:.1f} ms / direct {got['fast_write_ms']:.1f} ms, "
          f"DOM read {got['dom_read_ms']:.1f} ms / direct {got['fast_read_ms']:.1f} ms")


@needs_bin
def test_model_file_reader_writer_on_reference_bytes(golden, tmp_path):
    """CPU: a model file written by the REFERENCE (oracle/_ref, the C1 500/6/5 forest) read by
    Forest::load's direct reader and written back by b200::json_write gives the very same
    bytes (and the reference's own DOM route agrees) -- the drop-in's model I/O path."""
    import ctypes as C
    os.environ.setdefault("AIWC_REF_QUARANTINE", "1")  # deterministic multi-threaded fit
    from oracle_lib import Ref, RefData, RefForest
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    L = Ref.lib()
    d = RefData()
    f = RefForest.fit(d, 500, 6, 5, golden["forest_seed"], jobs=8)
    L.ref_forest_json.restype = C.c_uint64
    L.ref_forest_json.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64]
    n = L.ref_forest_json(f.h, None, 0)
    buf = C.create_string_buffer(n)
    L.ref_forest_json(f.h, buf, n)
    path = tmp_path / "c1_500.json"
    path.write_bytes(buf.raw[:n])
    r = subprocess.run([BIN, "jsonfile", str(path)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr + r.stdout
    got = json.loads(r.stdout.strip().splitlines()[-1])
    assert got["identical"] is True and got["bytes"] == C1_JSON_SIZE + 1
    assert got["fnv"] == golden["c1_500_6_5"]["json_fnv_with_newline"]
