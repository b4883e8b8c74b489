"""Pin the CPU oracle (oracle/) against golden vectors produced by the REAL
reference (oracle/make_golden.py imports ringacc).  CPU only."""
import json

import numpy as np
import pytest

from .conftest import GOLDEN


def test_generator_matches_reference(golden, oracle):
    g = golden("gen.npz")
    n_cases = len([k for k in g.files if k.endswith("_meta")])
    assert n_cases >= 7
    for i in range(n_cases):
        seed, _sub, _rank, lane, meas, wr, nk, nw, mode = (int(x) for x in g[f"c{i}_meta"])
        up, down = oracle.gsigma(seed, wr, lane, meas, nk * nw, "float" if mode == 0 else "integer")
        if mode == 1:  # integer lattice: bitwise
            assert np.array_equal(up, g[f"c{i}_up"]) and np.array_equal(down, g[f"c{i}_down"])
        else:  # float: sin/cos implementations may differ by an ulp across hosts
            np.testing.assert_allclose(up, g[f"c{i}_up"], rtol=0, atol=1e-15)
            np.testing.assert_allclose(down, g[f"c{i}_down"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("impl", ["c", "numpy"])
def test_accumulate_matches_reference_bitwise(golden, oracle, impl):
    a = golden("acc.npz")
    fn = oracle.accumulate if impl == "c" else oracle.accumulate_np
    for i in range(len([k for k in a.files if k.endswith("_meta")])):
        nk, nw, lo, hi, nwalk = (int(x) for x in a[f"c{i}_meta"])
        g4 = a[f"c{i}_start"].copy()
        for w in range(nwalk):
            fn(g4, lo, hi, a[f"c{i}_up"][w], a[f"c{i}_down"][w])
        # bitwise: same per-entry op order as numpy's complex ops on an FMA host
        assert np.array_equal(g4, a[f"c{i}_end"]), f"case {i} (N={nk * nw}, [{lo},{hi}))"


def test_config1_golden(golden, oracle):
    c1 = golden("c1.npz")
    for key in c1.files:
        mode, seed = key.split("_")
        g4 = np.zeros((1, 32, 32), np.complex128)
        for w in range(16):
            up, down = oracle.gsigma(int(seed), 0, w, 0, 32, mode)
            oracle.accumulate(g4, 0, 1, up, down)
        if mode == "integer":
            assert np.array_equal(g4, c1[key])
        else:
            np.testing.assert_allclose(g4, c1[key], rtol=1e-13, atol=1e-13)


def test_serial_oracle_golden(golden, oracle):
    o = golden("oracle.npz")
    for i in range(len([k for k in o.files if k.endswith("_meta")])):
        seed, s, S, k, m, nk, nw, mode = (int(x) for x in o[f"c{i}_meta"])
        mode = "float" if mode == 0 else "integer"
        out = oracle.oracle_full(seed, nk * nw, s, S, k, m, mode)
        if mode == "integer":
            assert np.array_equal(out, o[f"c{i}_tensor"])
        else:
            np.testing.assert_allclose(out, o[f"c{i}_tensor"], rtol=1e-13, atol=1e-13)


def test_brute_force_agrees(oracle):
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 4, 6):
        up = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        down = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        g4 = np.zeros((n, n, n), np.complex128)
        oracle.accumulate(g4, 0, n, up, down)
        np.testing.assert_allclose(g4, oracle.brute_force(up, down, 0, n), rtol=1e-14, atol=1e-14)


def test_index_and_partition_known_answers(oracle):
    misc = json.loads((GOLDEN / "misc.json").read_text())
    for a, b, n, want in misc["index_diff"]:
        assert oracle.index_diff(a, b, n) == want
    for n, p, ranges in misc["partition"]:
        assert [list(r) for r in oracle.partition(n, p)] == ranges


def test_c64_oracle_close_to_c128(oracle):
    rng = np.random.default_rng(5)
    n = 12
    up = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
    down = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
    a = np.zeros((3, n, n), np.complex128)
    b = np.zeros((3, n, n), np.complex64)
    oracle.accumulate(a, 4, 7, up, down)
    oracle.accumulate(b, 4, 7, up, down)
    assert oracle.compare(a, b)["l2_real"] < 1e-6


def test_accuracy_metrics_match_reference_definitions():
    """paper_2105_00027_b200.accuracy restates ringacc.accuracy's metrics
    (accuracy.py:23-64) on numpy or torch tensors (CPU here)."""
    import numpy as np
    import pytest as _pt
    from paper_2105_00027_b200 import accuracy as A
    rng = np.random.default_rng(3)
    ref = rng.standard_normal((3, 4, 4)) + 1j * rng.standard_normal((3, 4, 4))
    test = ref + 1e-9 * (rng.standard_normal(ref.shape) + 1j * rng.standard_normal(ref.shape))
    r = A.compare(ref, test)
    want_l1 = np.abs(ref.real - test.real).sum() / np.abs(ref.real).sum()
    want_l2 = np.sqrt((np.abs(ref.imag - test.imag) ** 2).sum() / (np.abs(ref.imag) ** 2).sum())
    assert r.l1_real == _pt.approx(want_l1, rel=1e-12) and r.l2_imag == _pt.approx(want_l2, rel=1e-12)
    assert r.passed and A.compare(ref, ref).to_dict()["pass"]
    bad = test.copy()
    bad.flat[0] += 1 + 1j
    assert not A.compare(ref, bad).passed
    with _pt.raises(A.UndefinedNormError):
        A.l1_error(np.zeros(4), np.ones(4))
