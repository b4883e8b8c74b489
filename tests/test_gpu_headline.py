"""Parity of the paths the bench headline and the BASELINE configs actually run,
at their own shapes ("Next round" item 1).  GPU only.

* the fused default (G4_ARITH_FUSED: the persistent K1 v3 with its TMEM
  hand-off and TMA tensor-reduce epilogue) on the full N = 512 x 64-plane x
  B = 8 bench workload, on a zero and on a nonzero slice;
* config 4's per-GPU share (N = 4608, 72 planes) through the multi-plane
  kernel, exact and fused, sampled planes of ONE 72-plane slice;
* config 3's index space (N = 1024, n_k = 16, n_w = 64), 16 planes;
* the 8-plane share of an 8-GPU ring (P = 8) in fused mode;
* B = 40 fused (more walkers than one launch takes: TMA_MAXW chunking);
* the reference-layout C entry ``g4_accumulate`` (K2 + K1 through a caller
  workspace) for G4_C128, G4_C64 and G4_C128_G64 with 70 walkers
  (> G4_MAX_BATCH = 64: two chunks).

The semantics matched are ringacc/tensor.py:233-251.  Tolerances: integer
payloads bitwise in every mode; float payloads bitwise in exact mode and within
1e-12 relative (complex128) / 1e-5 (complex64) in fused mode -- tighter than
north_star's 1e-10 / 1e-5.
"""
import ctypes

import numpy as np
import pytest
import torch

from paper_2105_00027_b200 import _lib
from paper_2105_00027_b200 import tensor as T

pytestmark = pytest.mark.gpu


def to_np(t):
    return t.detach().cpu().numpy()


@pytest.fixture
def fused():
    lib = _lib.load()
    _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED))
    yield lib
    _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_EXACT))


def k1_config(n, planes, nb, dtype=_lib.G4_C128):
    out = (ctypes.c_int32 * 9)()
    _lib.check(_lib.load().g4_k1_config(n, planes, nb, dtype, out))
    return list(out)


def _walkers(sp, seed, mode, nb, dtype=torch.complex128, dev=None):
    return [T.generate_gsigma(seed, T.Origin(0, 0, w, 0, 0), sp, mode, device=dev, dtype=dtype)
            for w in range(nb)]


def _check(got, ref, mode, tol):
    if mode == "integer" or tol == 0.0:
        assert np.array_equal(got, ref)
    else:
        np.testing.assert_allclose(got, ref, rtol=tol, atol=tol * np.abs(ref).max())


@pytest.mark.parametrize("start", ["zero", "nonzero"])
def test_headline_fused_full_slice(oracle, cuda_dev, fused, start):
    """The bench default: N = 512, all 64 planes, 8 walkers, one fused pass --
    every entry checked (the deferred update adds the walkers' sum to the slice
    in L2, so the nonzero start matters)."""
    sp = T.CombinedIndexSpace(16, 32)
    n, planes, B = sp.size, 64, 8
    cfg = k1_config(n, planes, B)
    assert cfg[0] == 3 and cfg[8] == 1, f"headline is not the persistent deferred kernel (v3): {cfg}"
    rng = np.random.default_rng(7)
    for mode in ("integer", "float"):
        if start == "zero":
            init = np.zeros((planes, n, n), np.complex128)
        else:
            init = (rng.integers(-3, 4, (planes, n, n)) + 1j * rng.integers(-3, 4, (planes, n, n))).astype(
                np.complex128)
        sl = T.GtSlice(sp, 0, planes, torch.from_numpy(init.copy()).to(cuda_dev))
        gs = _walkers(sp, 0, mode, B, dev=cuda_dev)
        T.accumulate_g4_batch(sl, gs)
        ref = init.copy()
        for g in gs:
            oracle.accumulate(ref, 0, planes, to_np(g.up.contiguous()), to_np(g.down.contiguous()))
        got = to_np(sl.data)
        _check(got, ref, mode, 1e-12)
        assert sl.meas_count == B


def test_headline_fused_repeatable(cuda_dev, fused):
    """Timing-dependent races would show as run-to-run differences: three fused
    passes from the same inputs must agree entry for entry (integer payloads)."""
    sp = T.CombinedIndexSpace(16, 32)
    n, planes = sp.size, 64
    gs = _walkers(sp, 1, "integer", 8, dev=cuda_dev)
    outs = []
    for _ in range(3):
        sl = T.GtSlice.zeros(sp, 0, planes, device=cuda_dev)
        T.accumulate_g4_batch(sl, gs)
        outs.append(sl.data.clone())
    assert all(torch.equal(outs[0], o) for o in outs[1:])


@pytest.mark.parametrize("arith", ["exact", "fused"])
def test_config4_share_sampled_planes(oracle, cuda_dev, arith):
    """Config 4's per-GPU share: one 72-plane slice at N = 4608 (24.5 GB) through
    the multi-plane kernel; first, middle and last planes vs the C oracle."""
    lib = _lib.load()
    _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED if arith == "fused" else _lib.G4_ARITH_EXACT))
    try:
        sp = T.CombinedIndexSpace(36, 128)
        n, lo, hi = sp.size, 144, 216
        B = 8 if arith == "fused" else 4  # fused: v3 from 8 walkers a pass (geometry 43 at this N)
        assert k1_config(n, hi - lo, B)[0] == (3 if arith == "fused" else 2)
        gs = _walkers(sp, 3, "float", B, dev=cuda_dev)
        sl = T.GtSlice.zeros(sp, lo, hi, device=cuda_dev)
        T.accumulate_g4_batch(sl, gs)
        torch.cuda.synchronize()
        host = [(to_np(g.up.contiguous()), to_np(g.down.contiguous())) for g in gs]
        del gs
        for q in (lo, lo + 37, hi - 1):
            ref = np.zeros((1, n, n), np.complex128)
            for up, down in host:
                oracle.accumulate(ref, q, q + 1, up, down)
            got = to_np(sl.data[q - lo:q - lo + 1])
            _check(got, ref, "float", 0.0 if arith == "exact" else 1e-12)
        del sl
        torch.cuda.empty_cache()
    finally:
        _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_EXACT))


@pytest.mark.parametrize("arith", ["exact", "fused"])
def test_config3_index_space(oracle, cuda_dev, arith):
    """Config 3's index space (n_k = 16, n_w = 64, N = 1024): the 16-plane share
    of one GPU in a sub-ring of 4, 8 walkers, every entry."""
    lib = _lib.load()
    _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED if arith == "fused" else _lib.G4_ARITH_EXACT))
    try:
        sp = T.CombinedIndexSpace(16, 64)
        n, lo, hi, B = sp.size, 16, 32, 8
        for mode in ("integer", "float"):
            gs = _walkers(sp, 5, mode, B, dev=cuda_dev)
            sl = T.GtSlice.zeros(sp, lo, hi, device=cuda_dev)
            T.accumulate_g4_batch(sl, gs)
            ref = np.zeros((hi - lo, n, n), np.complex128)
            for g in gs:
                oracle.accumulate(ref, lo, hi, to_np(g.up.contiguous()), to_np(g.down.contiguous()))
            _check(to_np(sl.data), ref, mode, 0.0 if arith == "exact" else 1e-12)
    finally:
        _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_EXACT))


def test_eight_gpu_share_fused(oracle, cuda_dev, fused):
    """P = 8 planes (config 2's per-GPU share on 8 GPUs), fused with deferral."""
    sp = T.CombinedIndexSpace(16, 32)
    n, lo, hi, B = sp.size, 40, 48, 8
    assert k1_config(n, hi - lo, B)[8] == 1
    for mode in ("integer", "float"):
        gs = _walkers(sp, 2, mode, B, dev=cuda_dev)
        sl = T.GtSlice.zeros(sp, lo, hi, device=cuda_dev)
        T.accumulate_g4_batch(sl, gs)
        ref = np.zeros((hi - lo, n, n), np.complex128)
        for g in gs:
            oracle.accumulate(ref, lo, hi, to_np(g.up.contiguous()), to_np(g.down.contiguous()))
        _check(to_np(sl.data), ref, mode, 1e-12)


@pytest.mark.parametrize("dtype", ["c128", "mixed", "c64"])
def test_many_walkers_fused(oracle, cuda_dev, fused, dtype):
    """B = 40 in one call: two launches of at most 32 walkers (tensor maps per
    launch), the second adding onto the first's deferred result."""
    sp = T.CombinedIndexSpace(8, 32)
    n, lo, hi, B = sp.size, 100, 132, 40
    gdt = torch.complex128 if dtype == "c128" else torch.complex64
    sdt = torch.complex64 if dtype == "c64" else torch.complex128
    for mode in ("integer", "float"):
        gs = _walkers(sp, 9, mode, B, dtype=gdt, dev=cuda_dev)
        sl = T.GtSlice.zeros(sp, lo, hi, device=cuda_dev, dtype=sdt)
        T.accumulate_g4_batch(sl, gs)
        ref = np.zeros((hi - lo, n, n), np.complex128)
        for g in gs:
            oracle.accumulate(ref, lo, hi, to_np(g.up.contiguous()).astype(np.complex128),
                              to_np(g.down.contiguous()).astype(np.complex128))
        if dtype == "c64":  # complex64 slices: 1e-5 (north_star); integer payloads exact
            got = to_np(sl.data).astype(np.complex128)
            if mode == "integer":
                assert np.array_equal(got, ref)
            else:
                np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-5 * np.abs(ref).max())
        else:
            _check(to_np(sl.data), ref, mode, 1e-12)


@pytest.mark.parametrize("dtype", [_lib.G4_C128, _lib.G4_C64, _lib.G4_C128_G64])
@pytest.mark.parametrize("arith", ["exact", "fused"])
def test_reference_layout_entry(oracle, cuda_dev, dtype, arith):
    """g4_accumulate (SURVEY 8b's named export, the bench's e2e path): reference
    -layout up/down device matrices, K2 into the caller's workspace, K1; 70
    walkers (two chunks of <= 64).  G4_C128_G64 rounds the complex128 inputs to
    complex64 payloads, so the oracle applies the rounded matrices."""
    lib = _lib.load()
    _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED if arith == "fused" else _lib.G4_ARITH_EXACT))
    try:
        n, lo, hi, B = 96, 10, 42, 70
        sp = T.CombinedIndexSpace(4, 24)
        sdt = torch.complex64 if dtype == _lib.G4_C64 else torch.complex128
        in_dt = torch.complex64 if dtype == _lib.G4_C64 else torch.complex128
        for mode in ("integer", "float"):
            mats = [T.generate_reference_layout(11, T.Origin(0, 0, w, 0, 0), sp, mode, device=cuda_dev,
                                                dtype=in_dt) for w in range(B)]
            ws_bytes = lib.g4_accumulate_workspace_bytes(n, B, dtype)
            assert ws_bytes > 0
            ws = torch.empty(ws_bytes, dtype=torch.uint8, device=cuda_dev)
            rng = np.random.default_rng(3)
            init = (rng.integers(-3, 4, (hi - lo, n, n)) + 1j * rng.integers(-3, 4, (hi - lo, n, n)))
            g4 = torch.from_numpy(init.astype(np.complex128)).to(cuda_dev).to(sdt)
            st = torch.cuda.current_stream(cuda_dev).cuda_stream
            _lib.check(lib.g4_accumulate(g4.data_ptr(), lo, hi, n,
                                         _lib.ptr_array([u.data_ptr() for u, _ in mats]),
                                         _lib.ptr_array([d.data_ptr() for _, d in mats]), B, dtype,
                                         _lib.G4_CHANNEL_EQ1, ws.data_ptr(), ws_bytes, st))
            torch.cuda.synchronize()
            ref = init.astype(np.complex128)
            for u, d in mats:
                uh, dh = to_np(u), to_np(d)
                if dtype == _lib.G4_C128_G64:
                    uh, dh = uh.astype(np.complex64), dh.astype(np.complex64)
                oracle.accumulate(ref, lo, hi, uh.astype(np.complex128), dh.astype(np.complex128))
            got = to_np(g4).astype(np.complex128)
            if dtype == _lib.G4_C64:
                _check(got, ref, mode if mode == "integer" else "float", 1e-5)
            else:
                _check(got, ref, mode, 0.0 if arith == "exact" else 1e-12)
    finally:
        _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_EXACT))


def test_reference_layout_entry_rejects_small_workspace(cuda_dev):
    lib = _lib.load()
    n = 64
    g4 = torch.zeros((4, n, n), dtype=torch.complex128, device=cuda_dev)
    u = torch.zeros((n, n), dtype=torch.complex128, device=cuda_dev)
    need = lib.g4_accumulate_workspace_bytes(n, 2, _lib.G4_C128)
    ws = torch.empty(need - 16, dtype=torch.uint8, device=cuda_dev)
    with pytest.raises(Exception) as e:
        _lib.check(lib.g4_accumulate(g4.data_ptr(), 0, 4, n, _lib.ptr_array([u.data_ptr()] * 2),
                                     _lib.ptr_array([u.data_ptr()] * 2), 2, _lib.G4_C128, _lib.G4_CHANNEL_EQ1,
                                     ws.data_ptr(), need - 16, 0))
    assert type(e.value).__name__ == "ContractViolation"


@pytest.mark.parametrize("geom", ["40", "43", "25", "27", "12", "13", "19"])
def test_forced_geometry_parity_repeated(geom):
    """Each production (and selectable warp-specialised) geometry forced on the
    small-slice suite AND the full N = 512 x 64 x 8 bench shape, exact and
    fused, three times (geometry 25's exact-mode race must not come
    back unnoticed).  Runs tools/geom_check.py in a subprocess because the
    geometry is read from the environment once per process."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, G4RING_V2GEOM=geom)
    r = subprocess.run([sys.executable, str(root / "tools" / "geom_check.py"), "--repeat", "3"], env=env,
                       cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count(" ok") == 3 * 24 and "MISMATCH" not in r.stdout
