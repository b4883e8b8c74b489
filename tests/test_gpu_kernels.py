"""Parity of the CUDA kernels (called through the C ABI via the mirror API)
against the CPU oracle and the reference's golden vectors.  GPU only.

Tolerances: complex128 results are BITWISE equal to the oracle (the kernel
uses the reference's exact op order); complex64 results are bitwise equal to
the binary32 oracle and within 1e-5 relative of the complex128 reference
(north_star); float-mode payloads generated ON THE DEVICE differ from numpy's
by <= 2 ulp (device sin/cos), so those comparisons use atol 1e-15 per entry.
"""
import numpy as np
import pytest
import torch

from paper_2105_00027_b200 import _lib
from paper_2105_00027_b200 import tensor as T
from paper_2105_00027_b200.errors import ContractViolation

pytestmark = pytest.mark.gpu


def to_np(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def payload(up, down, dev, dtype=torch.complex128):
    n = up.shape[0]
    return T.GSigma(T.CombinedIndexSpace(1, n), up, down, device=dev, dtype=dtype)


def test_accumulate_matches_reference_golden(golden, cuda_dev):
    a = golden("acc.npz")
    for i in range(len([k for k in a.files if k.endswith("_meta")])):
        nk, nw, lo, hi, nwalk = (int(x) for x in a[f"c{i}_meta"])
        sp = T.CombinedIndexSpace(nk, nw)
        sl = T.GtSlice(sp, lo, hi, torch.from_numpy(a[f"c{i}_start"]).to(cuda_dev))
        gs = [T.GSigma(sp, a[f"c{i}_up"][w], a[f"c{i}_down"][w], device=cuda_dev) for w in range(nwalk)]
        for g in gs:
            T.accumulate_g4(sl, g)
        assert np.array_equal(to_np(sl.data), a[f"c{i}_end"]), f"case {i}"
        assert sl.meas_count == int(a[f"c{i}_count"])
        # the batched form is bitwise identical to sequential calls
        sl2 = T.GtSlice(sp, lo, hi, torch.from_numpy(a[f"c{i}_start"]).to(cuda_dev))
        T.accumulate_g4_batch(sl2, gs)
        assert torch.equal(sl.data, sl2.data)


@pytest.mark.parametrize("n,lo,hi,nb", [(64, 0, 64, 1), (64, 13, 29, 3), (96, 90, 96, 5),
                                        (33, 0, 33, 17), (128, 64, 72, 70), (5, 1, 4, 2),
                                        (1, 0, 1, 3), (2, 0, 2, 4), (3, 2, 3, 9)])
def test_random_shapes_bitwise_vs_oracle(oracle, cuda_dev, n, lo, hi, nb):
    rng = np.random.default_rng(n * 1000 + lo)
    start = rng.standard_normal((hi - lo, n, n)) + 1j * rng.standard_normal((hi - lo, n, n))
    ref = start.copy()
    sp = T.CombinedIndexSpace(1, n)
    sl = T.GtSlice(sp, lo, hi, torch.from_numpy(start).to(cuda_dev))
    gs = []
    for _ in range(nb):
        up = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
        down = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
        oracle.accumulate(ref, lo, hi, up, down)
        gs.append(T.GSigma(sp, up, down, device=cuda_dev))
    T.accumulate_g4_batch(sl, gs)  # > G4_MAX_BATCH walkers are chunked in order
    assert np.array_equal(to_np(sl.data), ref)


@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("n,lo,hi,nb", [(64, 3, 64, 9), (100, 0, 17, 4), (257, 250, 257, 6),
                                        (512, 500, 512, 5), (200, 0, 5, 3), (67, 60, 67, 2)])
def test_both_kernel_variants_bitwise(oracle, cuda_dev, variant, n, lo, hi, nb):
    lib = _lib.load()
    _lib.check(lib.g4_set_kernel_variant(variant))
    try:
        test_random_shapes_bitwise_vs_oracle(oracle, cuda_dev, n, lo, hi, nb)
    finally:
        _lib.check(lib.g4_set_kernel_variant(0))


def test_config1_device_generator(golden, cuda_dev):
    """BASELINE config 1: N=32, K3={0}, 16 walkers generated on the device."""
    c1 = golden("c1.npz")
    sp = T.CombinedIndexSpace(4, 8)
    for key in c1.files:
        mode, seed = key.split("_")
        sl = T.GtSlice.zeros(sp, 0, 1, device=cuda_dev)
        gs = [T.generate_gsigma(int(seed), T.Origin(0, 0, w, 0, 0), sp, mode, device=cuda_dev)
              for w in range(16)]
        T.accumulate_g4_batch(sl, gs)
        got = to_np(sl.data)
        if mode == "integer":
            assert np.array_equal(got, c1[key])
        else:
            np.testing.assert_allclose(got, c1[key], rtol=1e-10, atol=1e-13)
        assert sl.meas_count == 16


@pytest.mark.parametrize("mode", ["integer", "float"])
def test_generator_vs_oracle(oracle, cuda_dev, mode):
    for (seed, wr, lane, meas, nk, nw) in [(0, 0, 0, 0, 2, 2), (1234, 9, 3, 4, 4, 8),
                                           (2**40 + 3, 7, 5, 999, 3, 5), (11, 1, 0, 2, 16, 32)]:
        sp = T.CombinedIndexSpace(nk, nw)
        ref_up, ref_down = oracle.gsigma(seed, wr, lane, meas, sp.size, mode)
        g = T.generate_gsigma(seed, T.Origin(0, 0, lane, meas, wr), sp, mode, device=cuda_dev)
        up, down = to_np(g.up), to_np(g.down)
        ru, rd = T.generate_reference_layout(seed, T.Origin(0, 0, lane, meas, wr), sp, mode,
                                             device=cuda_dev)
        if mode == "integer":
            assert np.array_equal(up, ref_up) and np.array_equal(down, ref_down)
            assert np.array_equal(to_np(ru), ref_up) and np.array_equal(to_np(rd), ref_down)
        else:
            for x, y in ((up, ref_up), (down, ref_down), (to_np(ru), ref_up), (to_np(rd), ref_down)):
                np.testing.assert_allclose(x, y, rtol=0, atol=1e-15)


def test_prepare_is_exact_transpose(cuda_dev):
    rng = np.random.default_rng(1)
    for n in (1, 7, 32, 33, 100):
        up = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        down = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        g = payload(up, down, cuda_dev)
        st = to_np(g.staged)
        assert st.shape == T.staged_shape(n, torch.complex128)
        assert np.array_equal(st[0, :n, :n], up.T) and np.array_equal(st[1, :n, :n], down.T)
        rr, cc = np.meshgrid(np.arange(st.shape[1]) % n, np.arange(st.shape[2]) % n, indexing="ij")
        assert np.array_equal(st[0], up.T[rr, cc]) and np.array_equal(st[1], down.T[rr, cc])  # halo
        assert np.array_equal(to_np(g.up.contiguous()), up)


def test_identity_known_answer(cuda_dev):
    """Both spins = I: every plane gains 2 on its K1 == K2 diagonal."""
    for n in (2, 5, 40):
        sp = T.CombinedIndexSpace(1, n)
        eye = np.eye(n, dtype=np.complex128)
        sl = T.GtSlice.zeros_full(sp, device=cuda_dev)
        T.accumulate_g4(sl, T.GSigma(sp, eye, eye, device=cuda_dev))
        expected = np.zeros((n, n, n), np.complex128)
        for k3 in range(n):
            expected[k3][np.diag_indices(n)] = 2
        assert np.array_equal(to_np(sl.data), expected)


def test_zero_payload_only_bumps_count(cuda_dev):
    sp = T.CombinedIndexSpace(2, 2)
    sl = T.GtSlice.zeros_full(sp, device=cuda_dev)
    T.accumulate_g4(sl, T.GSigma.empty(sp, device=cuda_dev))
    assert int(torch.count_nonzero(sl.data)) == 0 and sl.meas_count == 1


def test_guard_planes_never_written(cuda_dev):
    sp = T.CombinedIndexSpace(2, 3)
    n = sp.size
    backing = torch.full((n, n, n), 99 + 99j, dtype=torch.complex128, device=cuda_dev)
    sl = T.GtSlice(sp, 2, 4, backing[2:4])
    T.accumulate_g4(sl, T.generate_gsigma(9, T.Origin(0, 0, 0, 0, 0), sp, device=cuda_dev))
    b = to_np(backing)
    for plane in (0, 1, 4, 5):
        assert np.all(b[plane] == 99 + 99j)
    assert not np.all(b[2] == 99 + 99j)


def test_guard_planes_large(cuda_dev):
    """Same at a kernel-relevant size: 4 owned planes inside 12, N=160."""
    sp = T.CombinedIndexSpace(16, 10)
    n = sp.size
    backing = torch.full((12, n, n), -7 + 3j, dtype=torch.complex128, device=cuda_dev)
    sl = T.GtSlice(sp, 5, 9, backing[4:8])
    gs = [T.generate_gsigma(3, T.Origin(0, 0, w, 0, 0), sp, device=cuda_dev) for w in range(5)]
    T.accumulate_g4_batch(sl, gs)
    b = to_np(backing)
    assert np.all(b[:4] == -7 + 3j) and np.all(b[8:] == -7 + 3j)


@pytest.mark.parametrize("n,p", [(6, 4), (12, 5), (64, 8)])
def test_slice_sum_equivalence(cuda_dev, n, p):
    """Per-slice accumulation over a partition stitches to the full tensor, bitwise."""
    sp = T.CombinedIndexSpace(1, n)
    gs = [T.generate_gsigma(17, T.Origin(0, 0, 0, m, 0), sp, "integer", device=cuda_dev) for m in range(3)]
    full = T.GtSlice.zeros_full(sp, device=cuda_dev)
    T.accumulate_g4_batch(full, gs)
    stitched = torch.zeros_like(full.data)
    for lo, hi in T.make_partition(n, p).ranges:
        sl = T.GtSlice.zeros(sp, lo, hi, device=cuda_dev)
        for g in gs:
            T.accumulate_g4(sl, g)
        stitched[lo:hi] = sl.data
    assert torch.equal(stitched, full.data)


def test_order_independent_in_integer_mode(cuda_dev):
    sp = T.CombinedIndexSpace(4, 4)
    a = T.generate_gsigma(1, T.Origin(0, 0, 0, 0, 0), sp, "integer", device=cuda_dev)
    b = T.generate_gsigma(1, T.Origin(0, 1, 0, 0, 1), sp, "integer", device=cuda_dev)
    ab, ba = T.GtSlice.zeros_full(sp, device=cuda_dev), T.GtSlice.zeros_full(sp, device=cuda_dev)
    T.accumulate_g4_batch(ab, [a, b])
    T.accumulate_g4_batch(ba, [b, a])
    assert torch.equal(ab.data, ba.data)


def test_contract_violations(cuda_dev):
    sp = T.CombinedIndexSpace(2, 2)
    g = T.generate_gsigma(0, T.Origin(0, 0, 0, 0, 0), sp, device=cuda_dev)
    with pytest.raises(ContractViolation):
        T.accumulate_g4(T.GtSlice.zeros_full(T.CombinedIndexSpace(2, 3), device=cuda_dev), g)
    with pytest.raises(ContractViolation):
        T.GtSlice.zeros(sp, 3, 3, device=cuda_dev)
    with pytest.raises(ContractViolation):
        T.accumulate_g4(T.GtSlice.zeros_full(sp, device=cuda_dev, dtype=torch.complex64), g)
    lib = _lib.load()
    sl = T.GtSlice.zeros_full(sp, device=cuda_dev)
    st = lib.g4_accumulate_staged(sl.data.data_ptr(), 0, 4, 4, _lib.ptr_array([g.staged.data_ptr()]),
                                  1, _lib.G4_C128, 7, None)
    with pytest.raises(ContractViolation, match="channel"):
        _lib.check(st)
    st = lib.g4_accumulate_staged(sl.data.data_ptr() + 8, 0, 4, 4,
                                  _lib.ptr_array([g.staged.data_ptr()]), 1, _lib.G4_C128, 0, None)
    with pytest.raises(ContractViolation, match="aligned"):
        _lib.check(st)


@pytest.mark.parametrize("n,lo,hi,variant", [(48, 10, 18, 0), (160, 5, 40, 0), (160, 5, 40, 1),
                                             (257, 240, 257, 2), (96, 0, 96, 2),
                                             (160, 3, 11, 0), (129, 120, 129, 0), (512, 0, 4, 0)])
def test_complex64(oracle, cuda_dev, n, lo, hi, variant):
    lib = _lib.load()
    _lib.check(lib.g4_set_kernel_variant(variant))
    try:
        _complex64_case(oracle, cuda_dev, n, lo, hi)
    finally:
        _lib.check(lib.g4_set_kernel_variant(0))


def _complex64_case(oracle, cuda_dev, n, lo, hi):
    rng = np.random.default_rng(8)
    sp = T.CombinedIndexSpace(1, n)
    ref128 = np.zeros((hi - lo, n, n), np.complex128)
    ref64 = np.zeros((hi - lo, n, n), np.complex64)
    sl = T.GtSlice.zeros(sp, lo, hi, device=cuda_dev, dtype=torch.complex64)
    gs = []
    for _ in range(6):
        up = (rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))).astype(np.complex64)
        down = (rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))).astype(np.complex64)
        oracle.accumulate(ref128, lo, hi, up.astype(np.complex128), down.astype(np.complex128))
        oracle.accumulate(ref64, lo, hi, up, down)
        gs.append(T.GSigma(sp, up, down, device=cuda_dev, dtype=torch.complex64))
    T.accumulate_g4_batch(sl, gs)
    got = to_np(sl.data)
    assert np.array_equal(got, ref64)
    np.testing.assert_allclose(got, ref128, rtol=1e-5, atol=1e-5 * np.abs(ref128).max())


def test_c128_payload_staged_as_c64(cuda_dev):
    rng = np.random.default_rng(2)
    n = 20
    up = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    down = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    g = payload(up, down, cuda_dev, dtype=torch.complex64)
    assert np.array_equal(to_np(g.staged)[0, :n, :n], up.T.astype(np.complex64))


def test_reduce_sum_canonical_order(cuda_dev):
    lib = _lib.load()
    rng = np.random.default_rng(4)
    srcs = [rng.standard_normal((3, 17, 17)) + 1j * rng.standard_normal((3, 17, 17)) for _ in range(5)]
    ts = [torch.from_numpy(s).to(cuda_dev) for s in srcs]
    dst = torch.empty_like(ts[0])
    _lib.check(lib.g4_reduce_sum(dst.data_ptr(), _lib.ptr_array([t.data_ptr() for t in ts]), 5,
                                 ts[0].numel(), _lib.G4_C128,
                                 torch.cuda.current_stream().cuda_stream))
    total = srcs[0].copy()
    for s in srcs[1:]:
        total += s  # base.py:135-148: rank order 0, 1, 2, ...
    assert np.array_equal(to_np(dst), total)


def test_flag_write_wait_single_process(cuda_dev):
    lib = _lib.load()
    flag = torch.zeros(2, dtype=torch.int64, device=cuda_dev)
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.g4_flag_write(flag.data_ptr(), 5, s))
    _lib.check(lib.g4_flag_wait(flag.data_ptr(), 5, s))
    torch.cuda.synchronize()
    assert int(flag[0]) == 5
    _lib.check(lib.g4_flag_host_wait(flag.data_ptr(), 5, 1000))
    with pytest.raises(Exception) as e:
        _lib.check(lib.g4_flag_host_wait(flag.data_ptr(), 6, 50))
    assert type(e.value).__name__ == "DeadlockError"


@pytest.mark.parametrize("n,planes", [(512, (0, 1, 63)), (4608, (0, 575))])
def test_full_size_sampled_planes(oracle, cuda_dev, n, planes):
    """BASELINE C2 / C4 index space sizes: sampled planes vs the C oracle, bitwise."""
    sp = T.CombinedIndexSpace(16 if n == 512 else 36, 32 if n == 512 else 128)
    gs = [T.generate_gsigma(0, T.Origin(0, 0, w, 0, 0), sp, "float", device=cuda_dev) for w in range(2)]
    host = [(to_np(g.up.contiguous()), to_np(g.down.contiguous())) for g in gs]
    for q in planes:
        sl = T.GtSlice.zeros(sp, q, q + 1, device=cuda_dev)
        T.accumulate_g4_batch(sl, gs)
        ref = np.zeros((1, n, n), np.complex128)
        for up, down in host:
            oracle.accumulate(ref, q, q + 1, up, down)
        assert np.array_equal(to_np(sl.data), ref), f"plane {q}"


@pytest.mark.parametrize("variant", [1, 2])
def test_fused_arith_within_tolerance(oracle, cuda_dev, variant):
    """G4_ARITH_FUSED: integer-valued payloads stay bitwise; float within 1e-12 relative."""
    lib = _lib.load()
    _lib.check(lib.g4_set_kernel_variant(variant))
    _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED))
    try:
        sp = T.CombinedIndexSpace(8, 16)
        n, lo, hi = sp.size, 30, 70
        for mode in ("integer", "float"):
            sl = T.GtSlice.zeros(sp, lo, hi, device=cuda_dev)
            gs = [T.generate_gsigma(5, T.Origin(0, 0, w, 0, 0), sp, mode, device=cuda_dev) for w in range(6)]
            T.accumulate_g4_batch(sl, gs)
            ref = np.zeros((hi - lo, n, n), np.complex128)
            for g in gs:
                oracle.accumulate(ref, lo, hi, to_np(g.up.contiguous()), to_np(g.down.contiguous()))
            got = to_np(sl.data)
            if mode == "integer":
                assert np.array_equal(got, ref)
            else:
                np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
                if variant == 1:  # v1 has no deferred update: fused mode runs the exact kernel
                    assert np.array_equal(got, ref)
                else:
                    assert not np.array_equal(got, ref)  # it really is the other evaluation order
    finally:
        _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_EXACT))
        _lib.check(lib.g4_set_kernel_variant(0))


@pytest.mark.parametrize("n,lo,hi,variant", [(40, 3, 9, 0), (128, 0, 40, 0), (128, 0, 40, 1), (161, 150, 161, 2),
                                             (161, 150, 161, 0), (96, 7, 15, 0)])
def test_mixed_precision_bitwise(oracle, cuda_dev, n, lo, hi, variant):
    """complex128 G4 with complex64 payloads: bitwise equal to the complex128
    reference applied to the complex64-rounded payloads (widening is exact)."""
    lib = _lib.load()
    _lib.check(lib.g4_set_kernel_variant(variant))
    try:
        rng = np.random.default_rng(n)
        sp = T.CombinedIndexSpace(1, n)
        start = rng.standard_normal((hi - lo, n, n)) + 1j * rng.standard_normal((hi - lo, n, n))
        ref = start.copy()
        sl = T.GtSlice(sp, lo, hi, torch.from_numpy(start).to(cuda_dev))
        gs = []
        for _ in range(5):
            up = (rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n)))
            down = (rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n)))
            gs.append(T.GSigma(sp, up, down, device=cuda_dev, dtype=torch.complex64))  # K2 rounds c128 -> c64
            oracle.accumulate(ref, lo, hi, up.astype(np.complex64).astype(np.complex128),
                              down.astype(np.complex64).astype(np.complex128))
        T.accumulate_g4_batch(sl, gs)
        assert np.array_equal(to_np(sl.data), ref)
    finally:
        _lib.check(lib.g4_set_kernel_variant(0))


@pytest.mark.parametrize("n,dtype", [(32, torch.complex128), (100, torch.complex128), (512, torch.complex128),
                                     (96, torch.complex64), (257, torch.complex64)])
def test_core_copy_plus_halo_rebuild_is_exact(cuda_dev, n, dtype):
    """The ring's wire format: g4_copy_payload_cores moves only the N x N cores
    of staged payloads, g4_fill_halo rebuilds the rest; together they give the
    staged payloads bit for bit."""
    lib = _lib.load()
    sp = T.CombinedIndexSpace(1, n)
    code = _lib.G4_C128 if dtype == torch.complex128 else _lib.G4_C64
    k = 3
    src = torch.empty((k,) + T.staged_shape(n, dtype), dtype=dtype, device=cuda_dev)
    for i in range(k):
        g = T.generate_gsigma(i, T.Origin(0, 0, i, 0, 0), sp, "float", device=cuda_dev, dtype=dtype)
        src[i].copy_(g.staged)
    dst = torch.full_like(src, complex(float("nan"), float("nan")))
    st = torch.cuda.current_stream(cuda_dev).cuda_stream
    _lib.check(lib.g4_copy_payload_cores(dst.data_ptr(), src.data_ptr(), k, n, code, st))
    _lib.check(lib.g4_fill_halo(_lib.ptr_array([dst[i].data_ptr() for i in range(k)]), k, n, code, st))
    torch.cuda.synchronize()
    assert torch.equal(torch.view_as_real(dst), torch.view_as_real(src))


@pytest.mark.parametrize("dtype,n,lo,hi,nb", [("c128", 96, 0, 40, 6), ("c64", 96, 3, 37, 5), ("mixed", 128, 0, 24, 8),
                                              ("c128", 128, 10, 18, 4), ("c128", 160, 0, 20, 3),
                                              # K1 v3 (>= 8 walkers, >= 16 planes) with a partial last column
                                              # strip and row wraps (the per-lane edge path), nonzero start
                                              ("c128", 200, 5, 45, 8), ("mixed", 150, 0, 33, 12),
                                              ("c128", 64, 0, 64, 9),
                                              # complex64 slices with >= 8 walkers (geometry 12, or v3's
                                              # complex64 kernel under G4RING_V3_C64=1)
                                              ("c64", 200, 0, 40, 9), ("c64", 128, 5, 37, 16)])
def test_fused_deferred_update(oracle, cuda_dev, dtype, n, lo, hi, nb):
    """G4_ARITH_FUSED with >= 3 walkers adds the walkers' sum to a NONZERO slice
    at the end (L2 reduction): integer payloads stay bitwise, float within
    1e-12 (c128, mixed) / 1e-5 (c64) relative."""
    lib = _lib.load()
    _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED))
    try:
        sp = T.CombinedIndexSpace(1, n)
        sdt = torch.complex64 if dtype == "c64" else torch.complex128
        gdt = torch.complex128 if dtype == "c128" else torch.complex64
        for mode in ("integer", "float"):
            rng = np.random.default_rng(n + nb)
            start = (rng.integers(-3, 4, (hi - lo, n, n)) + 1j * rng.integers(-3, 4, (hi - lo, n, n)))
            ref = start.astype(np.complex128)
            sl = T.GtSlice(sp, lo, hi, torch.from_numpy(start.astype(np.complex128)).to(cuda_dev).to(sdt))
            gs = [T.generate_gsigma(2, T.Origin(0, 0, w, 0, 0), sp, mode, device=cuda_dev, dtype=gdt)
                  for w in range(nb)]
            T.accumulate_g4_batch(sl, gs)
            for g in gs:
                oracle.accumulate(ref, lo, hi, to_np(g.up.contiguous()).astype(np.complex128),
                                  to_np(g.down.contiguous()).astype(np.complex128))
            got = to_np(sl.data).astype(np.complex128)
            if mode == "integer":
                assert np.array_equal(got, ref)
            else:
                tol = 1e-5 if dtype == "c64" else 1e-12
                np.testing.assert_allclose(got, ref, rtol=tol, atol=tol * np.abs(ref).max())
    finally:
        _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_EXACT))


def test_bench_workload_full_slice(oracle, cuda_dev):
    """The bench's own N = 1 workload, checked in full (size-independent property
    at BASELINE config 2 size): N = 512, all 64 exchange planes, one K1 pass of
    8 device-generated walkers through the production geometry.  Integer mode
    bitwise over every entry; float mode within 1e-13 of the numpy restatement
    (the reference's own arithmetic), and its checksum within 1e-12."""
    sp = T.CombinedIndexSpace(16, 32)
    n, planes, B = sp.size, 64, 8
    for mode in ("integer", "float"):
        sl = T.GtSlice.zeros(sp, 0, planes, device=cuda_dev)
        gs = [T.generate_gsigma(0, T.Origin(0, 0, w, 0, 0), sp, mode, device=cuda_dev) for w in range(B)]
        T.accumulate_g4_batch(sl, gs)
        ref = np.zeros((planes, n, n), np.complex128)
        for g in gs:
            oracle.accumulate_np(ref, 0, planes, to_np(g.up.contiguous()), to_np(g.down.contiguous()))
        got = to_np(sl.data)
        if mode == "integer":
            assert np.array_equal(got, ref)
        else:
            scale = np.abs(ref).max()
            np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-13 * scale)
            assert abs(got.sum() - ref.sum()) <= 1e-12 * np.abs(ref).sum()


def test_cluster_multicast_geometry_parity():
    """Geometry 22 (geometry 12 in 2-CTA clusters sharing the shifted band by TMA
    multicast; selectable, not a default) against the C oracle: exact bitwise,
    fused within 1e-12, including the N % 32 != 0 fallback (tools/geom_check.py)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, G4RING_V2GEOM="22")
    r = subprocess.run([sys.executable, str(root / "tools" / "geom_check.py")], env=env, cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count(" ok") == 24


@pytest.mark.parametrize("arith,dtype,n_k,n_w,planes,nb,geom", [
    ("fused", "c128", 16, 32, 64, 8, 40),    # the headline: K1 v3
    ("fused", "mixed", 16, 32, 64, 8, 40),
    ("fused", "c128", 48, 48, 16, 8, 43),    # N > 2048: v3 with 10 park slots
    ("fused", "c128", 16, 32, 64, 5, 25),    # 4-7 walkers: geometry 25
    ("fused", "c128", 16, 32, 64, 2, 13),    # < 3 walkers: the exact kernel
    ("exact", "c128", 16, 32, 64, 8, 13),
    ("fused", "c64", 16, 32, 64, 8, 12),
    ("fused", "c128", 16, 32, 8, 8, 19),     # the 8-GPU share of config 2
    ("exact", "c128", 16, 32, 2, 8, 1),      # v1
])
def test_dispatch_launches_the_reported_kernel(cuda_dev, arith, dtype, n_k, n_w, planes, nb, geom):
    """The kernel a launch actually runs (g4_last_k1_geometry) is the one the
    selection table names -- a dispatch slip would stay
    invisible to the parity tests, which every kernel passes."""
    lib = _lib.load()
    _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED if arith == "fused" else _lib.G4_ARITH_EXACT))
    try:
        sp = T.CombinedIndexSpace(n_k, n_w)
        sdt = torch.complex64 if dtype == "c64" else torch.complex128
        gdt = torch.complex128 if dtype == "c128" else torch.complex64
        sl = T.GtSlice.zeros(sp, 0, planes, device=cuda_dev, dtype=sdt)
        gs = [T.GSigma.empty(sp, device=cuda_dev, dtype=gdt) for _ in range(nb)]
        T.accumulate_g4_batch(sl, gs)
        torch.cuda.synchronize()
        assert lib.g4_last_k1_geometry() == geom
    finally:
        _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_EXACT))
