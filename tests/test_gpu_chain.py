"""Chained fused passes (g4_k1.cuh, k1_chain_prev): back-to-back K1 v3 fused
launches on one stream overlap -- a pass does not wait for the previous one
before its payload loads and slice reductions, only before it exits.  These
tests issue passes with no synchronisation in between (pre-staged payloads, so
the stream holds nothing but K1 launches) and check the slice against the C
oracle: bitwise for integer payloads (a lost or doubled reduction would show),
1e-12 relative for float payloads.  Exact passes in between must break the
chain (they load and store the slice).  Semantics: ringacc/tensor.py:233-251.
GPU only.
"""
import ctypes

import numpy as np
import pytest
import torch

from paper_2105_00027_b200 import _lib
from paper_2105_00027_b200 import tensor as T

pytestmark = pytest.mark.gpu


def _mode(lib, fused):
    _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED if fused else _lib.G4_ARITH_EXACT))


def _k1_config(n, planes, nb):
    out = (ctypes.c_int32 * 9)()
    _lib.check(_lib.load().g4_k1_config(n, planes, nb, _lib.G4_C128, out))
    return list(out)


def _walkers(sp, seed, mode, nb, dev):
    return [T.generate_gsigma(seed, T.Origin(0, 0, w, 0, 0), sp, mode, device=dev) for w in range(nb)]


def _oracle(oracle, init, planes, batches):
    ref = init.copy()
    for gs in batches:
        for g in gs:
            oracle.accumulate(ref, 0, planes, g.up.contiguous().cpu().numpy(), g.down.contiguous().cpu().numpy())
    return ref


@pytest.mark.parametrize("mode", ["integer", "float"])
def test_chained_fused_passes(oracle, cuda_dev, mode):
    """Five fused passes of 8 walkers on the bench shape (N = 512, 64 planes,
    v3), launched back to back on a nonzero slice."""
    lib = _lib.load()
    sp = T.CombinedIndexSpace(16, 32)
    n, planes = sp.size, 64
    _mode(lib, True)
    try:
        assert _k1_config(n, planes, 8)[0] == 3
        rng = np.random.default_rng(11)
        init = (rng.integers(-3, 4, (planes, n, n)) + 1j * rng.integers(-3, 4, (planes, n, n))).astype(np.complex128)
        batches = [_walkers(sp, 20 + i, mode, 8, cuda_dev) for i in range(5)]
        sl = T.GtSlice(sp, 0, planes, torch.from_numpy(init.copy()).to(cuda_dev))
        torch.cuda.synchronize()
        for gs in batches:
            T.accumulate_g4_batch(sl, gs)
        got = sl.data.cpu().numpy()
    finally:
        _mode(lib, False)
    ref = _oracle(oracle, init, planes, batches)
    if mode == "integer":
        assert np.array_equal(got, ref)
    else:
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def test_chain_broken_by_exact_passes(oracle, cuda_dev):
    """fused, fused, exact, fused, fused, exact, fused: the exact passes (v2,
    slice loads and stores) run between chained reductions; integer payloads,
    bitwise."""
    lib = _lib.load()
    sp = T.CombinedIndexSpace(8, 32)
    n, planes = sp.size, 64
    seq = [True, True, False, True, True, False, True]
    batches = [_walkers(sp, 40 + i, "integer", 8, cuda_dev) for i in range(len(seq))]
    sl = T.GtSlice.zeros(sp, 0, planes, device=cuda_dev)
    torch.cuda.synchronize()
    try:
        for fused, gs in zip(seq, batches):
            _mode(lib, fused)
            T.accumulate_g4_batch(sl, gs)
        got = sl.data.cpu().numpy()
    finally:
        _mode(lib, False)
    ref = _oracle(oracle, np.zeros((planes, n, n), np.complex128), planes, batches)
    assert np.array_equal(got, ref)


def test_chain_repeatable_many_passes(cuda_dev):
    """Twenty chained passes from the same inputs, twice: entry for entry equal
    (integer payloads), and equal to twenty times one pass."""
    lib = _lib.load()
    sp = T.CombinedIndexSpace(16, 32)
    planes = 64
    gs = _walkers(sp, 5, "integer", 8, cuda_dev)
    _mode(lib, True)
    try:
        outs = []
        for _ in range(2):
            sl = T.GtSlice.zeros(sp, 0, planes, device=cuda_dev)
            for _ in range(20):
                T.accumulate_g4_batch(sl, gs)
            outs.append(sl.data.clone())
        one = T.GtSlice.zeros(sp, 0, planes, device=cuda_dev)
        T.accumulate_g4_batch(one, gs)
    finally:
        _mode(lib, False)
    assert torch.equal(outs[0], outs[1])
    assert torch.equal(outs[0], one.data * 20)


@pytest.mark.parametrize("case", ["p8_geom19", "c64_geom12", "b5_geom25", "v2_v3_alternating"])
def test_chained_v2_deferred_passes(oracle, cuda_dev, case):
    """The v2 deferred kernels chain too (and with v3): P = 8 (the 8-GPU ring
    share), complex64 slices, 4-7 walkers a pass, and passes alternating
    between 5 walkers (v2 geometry 25) and 8 (v3); integer payloads, bitwise."""
    lib = _lib.load()
    sp = T.CombinedIndexSpace(16, 32)
    n = sp.size
    planes, sizes, dt = {
        "p8_geom19": (8, [8] * 6, torch.complex128),
        "c64_geom12": (64, [8] * 5, torch.complex64),
        "b5_geom25": (64, [5] * 5, torch.complex128),
        "v2_v3_alternating": (64, [5, 8, 5, 8, 8, 5], torch.complex128),
    }[case]
    batches = [[T.generate_gsigma(60 + i, T.Origin(0, 0, w, 0, 0), sp, "integer", device=cuda_dev, dtype=dt)
                for w in range(b)] for i, b in enumerate(sizes)]
    sl = T.GtSlice.zeros(sp, 0, planes, device=cuda_dev, dtype=dt)
    torch.cuda.synchronize()
    _mode(lib, True)
    try:
        for gs in batches:
            T.accumulate_g4_batch(sl, gs)
        got = sl.data.cpu().numpy().astype(np.complex128)
    finally:
        _mode(lib, False)
    ref = np.zeros((planes, n, n), np.complex128)
    for gs in batches:
        for g in gs:
            oracle.accumulate(ref, 0, planes, g.up.contiguous().cpu().numpy().astype(np.complex128),
                              g.down.contiguous().cpu().numpy().astype(np.complex128))
    assert np.array_equal(got, ref)
