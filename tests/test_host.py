"""CPU: host side of libaiwc_cuda.so -- the library loads without a GPU, exports every
symbol include/aiwc_cuda.h declares, its synthetic tables equal the reference's bit for
bit, and the host-side OOB finalisation matches the oracle.  No GPU compute here."""
import hashlib
import os
import re

import numpy as np
import pytest

import paper_1811_00156_b200 as pkg
from oracle_lib import Oracle, Ref, RefData

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "aiwc_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(aiwc_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = pkg.lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert L.aiwc_version().decode().startswith("aiwc-b200")


def test_no_cpu_fallback_without_gpu():
    if pkg.device_count() > 0:
        pytest.skip("GPU present")
    t = pkg.Table(3, 2)
    with pytest.raises(pkg.CudaError):
        pkg.PreparedDataset.from_table(t)


def test_derive_seed_matches_reference(golden):
    assert pkg.derive_seed(1, "forest") == golden["forest_seed"]
    assert pkg.derive_seed(7, "query", 12345) == Oracle.derive_seed(7, "query", 12345)


def test_synth_c1_matches_reference_golden(golden):
    t = pkg.Table()  # C1 defaults: 37 kernels, 15 devices, noise 0.02, seed 1
    g = golden["c1"]
    assert (t.n, t.p, t.fingerprint) == (g["n"], g["p"], g["fingerprint"])
    assert hashlib.sha256(t.col.tobytes() + t.y.tobytes()).hexdigest() == g["data_sha"]
    assert hashlib.sha256(t.seconds.tobytes()).hexdigest() == g["seconds_sha"]
    assert hashlib.sha256(t.kernel_of_row.tobytes()).hexdigest() == g["kernel_sha"]


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("K,D,noise,seed", [(11, 3, 0.0, 5), (120, 4, 0.1, 9), (5, 101, 0.02, 2)])
def test_synth_matches_reference_live(K, D, noise, seed):
    """kernel/device names >= 100 sort lexicographically (dataset.hpp:111-114)."""
    t = pkg.Table(K, D, noise, seed)
    r = RefData(K, D, noise, seed)
    assert (t.n, t.p, t.fingerprint) == (r.n, r.p, r.fingerprint)
    assert np.array_equal(t.col.view(np.uint64), r.col.view(np.uint64))
    assert np.array_equal(t.y.view(np.uint64), r.y.view(np.uint64))
    assert np.array_equal(t.seconds.view(np.uint64), r.seconds.view(np.uint64))
    assert np.array_equal(t.kernel_of_row, r.kernel)


@pytest.mark.slow
def test_synth_c4_matches_reference_golden(golden):
    t = pkg.Table(6757, 37)
    g = golden["c4"]
    assert (t.n, t.p, t.fingerprint) == (g["n"], g["p"], g["fingerprint"])
    assert hashlib.sha256(t.col.tobytes() + t.y.tobytes()).hexdigest() == g["data_sha"]


def test_oob_finalize_matches_oracle(golden):
    z = np.load(os.path.join(ROOT, "tests", "golden", "edge_ties.npz"))
    from oracle_lib import ForestSoA
    s = ForestSoA(z["offsets"], z["feature"], z["threshold"], z["left"], z["right"], z["value"],
                  inbag=z["inbag"])
    col, y = z["col"], z["y"]
    p, n = col.shape
    stats, rs, rc = Oracle.oob(col, y, n, p, s)
    st = pkg.oob_finalize(y, rs, rc)
    assert [st.degenerate, st.mse, st.response_variance, st.error_pct, st.r_squared,
            st.rows_evaluated] == list(stats)
    assert np.array_equal(stats, z["oob"])
    # constant response -> degenerate marker, no throw (forest.hpp:409-412)
    st2 = pkg.oob_finalize(np.ones(5), np.zeros(5), np.zeros(5, np.uint32))
    assert st2.degenerate
    with pytest.raises(pkg.ExecutionError):
        pkg.oob_finalize(np.arange(4.0), np.zeros(4), np.zeros(4, np.uint32))
