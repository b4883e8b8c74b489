"""The ring driver on the GPU: several rank processes (sharing the one B200 of
the test box, or one per GPU) connected through CUDA IPC peer memory, copy-
engine transfers and stream flags.  Compared with the oracle and with the
reference engine's golden outputs.  GPU only.

Tolerances: integer mode bitwise (any accumulation order); float mode 1e-10
relative (north_star: the ring reorders walkers).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2105_00027_b200 import engine as E
from paper_2105_00027_b200.errors import ConfigError, DeadlockError

pytestmark = pytest.mark.gpu


def cfg(**kw):
    base = dict(n_k=2, n_w=4, world_size=1, subring_size=1, lanes=1, measurements=2, seed=11,
                value_mode="integer", timeout_s=20.0)
    base.update(kw)
    return E.ExperimentConfig(**base)


def oracle_of(c):
    return O.oracle_full(c.seed, c.space_size, c.world_size // c.subring_size, c.subring_size, c.lanes,
                         c.measurements, c.value_mode, 0, c.num_planes)


def check(c, rep):
    ref = oracle_of(c)
    if c.value_mode == "integer":
        assert np.array_equal(rep.tensor, ref)
    else:
        np.testing.assert_allclose(rep.tensor, ref, rtol=1e-10, atol=1e-10 * np.abs(ref).max())
    s, k, m = c.subring_size, c.lanes, c.measurements
    steps = s - 1 if c.ring_steps_override is None else c.ring_steps_override
    for r in range(c.world_size):
        for t in range(k):
            cnt = rep.lane_counters[(r, t)]
            assert cnt.envelopes_sent == steps * m and cnt.envelopes_received == steps * m
            assert cnt.accumulations_applied == (steps + 1) * m
            origins = rep.lane_meta[(r, t)]["origins"]
            assert len(origins) == len(set(origins)) == (steps + 1) * m
            assert all(o[2] == t and o[0] == r // s for o in origins)
        assert rep.meas_counts[r] == (steps + 1) * m * k


@pytest.mark.parametrize("mode", ["integer", "float"])
def test_single_rank_is_serial_oracle(mode):
    c = cfg(value_mode=mode, measurements=5, lanes=2)
    check(c, E.run_experiment(c))


@pytest.mark.parametrize("kw", [
    dict(world_size=2, subring_size=2),
    dict(world_size=4, subring_size=4, lanes=2, measurements=3),
    dict(world_size=4, subring_size=2, lanes=1, measurements=2),          # 2 sub-rings + reduce
    dict(world_size=3, subring_size=3, lanes=3, direction="alternate", n_w=3),
    dict(world_size=4, subring_size=4, lanes=2, batch=2, measurements=5),  # batched rounds, partial last
    dict(world_size=4, subring_size=2, lanes=2, value_mode="float", n_k=8, n_w=16, planes=64),
])
def test_multi_rank_ring_matches_oracle(kw):
    c = cfg(**kw)
    check(c, E.run_experiment(c))


def test_reference_engine_golden(golden):
    """Same configs as the reference run_experiment golden outputs (engine.npz)."""
    e = golden("engine.npz")
    for i in (0, 2):
        nk, nw, world, s, lanes, m, seed = (int(x) for x in e[f"c{i}_cfg"])
        for mode in ("integer", "float"):
            c = cfg(n_k=nk, n_w=nw, world_size=world, subring_size=s, lanes=lanes, measurements=m,
                    seed=seed, value_mode=mode)
            rep = E.run_experiment(c)
            want = e[f"c{i}_{mode}_tensor"]
            if mode == "integer":
                assert np.array_equal(rep.tensor, want)
            else:
                np.testing.assert_allclose(rep.tensor, want, rtol=1e-10, atol=1e-12)
            assert [rep.slices[r] for r in range(world)] == [tuple(x) for x in e[f"c{i}_{mode}_slices"]]


def test_c64_ring_within_tolerance():
    c = cfg(world_size=2, subring_size=2, lanes=1, measurements=3, value_mode="float", dtype="c64",
            n_k=4, n_w=16)
    rep = E.run_experiment(c)
    ref = oracle_of(c)
    assert O.compare(ref, rep.tensor.astype(np.complex128))["l2_real"] < 1e-5


def test_mixed_precision_ring():
    c = cfg(world_size=2, subring_size=2, lanes=2, measurements=2, value_mode="float", dtype="c128g64",
            n_k=4, n_w=24, planes=40)
    rep = E.run_experiment(c)
    assert rep.tensor.dtype == np.complex128
    ref = oracle_of(c)
    r = O.compare(ref, rep.tensor)
    assert max(r["l1_real"], r["l1_imag"], r["l2_real"], r["l2_imag"]) < 1e-6  # c64-rounded payloads


def test_config4_scale_distributed_sampled_planes(oracle):
    """BASELINE config 4 index space (N = 4608): 2 ranks x 72 planes (the per-GPU
    share of the 8-GPU run, 49 GB of G4 in total) accumulated through the ring
    without gathering; sampled planes (first/last of each slice) vs the C oracle."""
    c = cfg(n_k=36, n_w=128, world_size=2, subring_size=2, lanes=1, measurements=1, value_mode="float",
            planes=144, gather=False, sample_planes=(0, 71, 72, 143), timeout_s=120.0, seed=3)
    rep = E.run_experiment(c)
    assert rep.tensor is None and set(rep.samples) == {0, 71, 72, 143}
    n = 4608
    walkers = [oracle.gsigma(c.seed, wr, 0, 0, n, "float") for wr in range(2)]
    for k3, got in rep.samples.items():
        ref = np.zeros((1, n, n), np.complex128)
        for up, down in walkers:
            oracle.accumulate(ref, k3, k3 + 1, up, down)
        np.testing.assert_allclose(got, ref[0], rtol=1e-10, atol=1e-13)


def test_short_ring_negative_control():
    c = cfg(world_size=3, subring_size=3, n_w=3, ring_steps_override=1)
    rep = E.run_experiment(c)
    assert rep.lane_counters[(0, 0)].envelopes_sent == 1 * 2
    assert rep.meas_counts[0] == 2 * 2
    assert not np.array_equal(rep.tensor, oracle_of(c))


def test_skipped_send_deadlocks_with_diagnostic():
    c = cfg(world_size=2, subring_size=2, measurements=1, fault="skip-send", timeout_s=3.0)
    with pytest.raises(DeadlockError) as err:
        E.run_experiment(c)
    msg = str(err.value)
    assert "rank 1" in msg and "lane 0" in msg and "step 0" in msg


def test_config_errors():
    with pytest.raises(ConfigError):
        E.validate_config(cfg(world_size=6, subring_size=4))
    with pytest.raises(ConfigError):
        E.validate_config(cfg(world_size=16, subring_size=16))  # more ranks than planes
    with pytest.raises(ConfigError):
        E.validate_config(cfg(lanes=1000))


def check_counts(c, rep):
    """Counter laws (C03) without origin tracking."""
    s, k, m = c.subring_size, c.lanes, c.measurements
    for r in range(c.world_size):
        for t in range(k):
            cnt = rep.lane_counters[(r, t)]
            assert cnt.envelopes_sent == (s - 1) * m and cnt.envelopes_received == (s - 1) * m
            assert cnt.accumulations_applied == s * m
        assert rep.meas_counts[r] == s * m * k


@pytest.mark.parametrize("kw", [
    dict(world_size=2, subring_size=2, measurements=8, batch=2),
    dict(world_size=4, subring_size=4, lanes=2, measurements=5),
    dict(world_size=4, subring_size=2, lanes=2, measurements=8, batch=2),      # sub-rings + reduce
    dict(world_size=3, subring_size=3, lanes=3, direction="alternate", n_w=3, measurements=5),
    dict(world_size=4, subring_size=4, lanes=1, value_mode="float", n_k=8, n_w=16, planes=64, measurements=16,
         batch=4),
    dict(world_size=4, subring_size=2, lanes=2, measurements=8, batch=2, lane_rings=True),  # per-lane pipelines
])
def test_native_round_program_matches_host_loop(kw, monkeypatch):
    """The native round program (one C call per round from round 2 on) against
    the per-op host loop on the same config (>= 4 rounds, so both round
    parities run natively): bitwise equal tensors (integer mode) or the same
    float result, and the same counters."""
    c = cfg(instrument=False, **kw)
    monkeypatch.setenv("G4RING_NATIVE", "1")
    native = E.run_experiment(c)
    monkeypatch.setenv("G4RING_NATIVE", "0")
    host = E.run_experiment(c)
    ref = oracle_of(c)
    if c.value_mode == "integer":
        assert np.array_equal(native.tensor, ref) and np.array_equal(host.tensor, ref)
    else:
        assert np.array_equal(native.tensor, host.tensor)  # same walkers in the same order per entry
        np.testing.assert_allclose(native.tensor, ref, rtol=1e-10, atol=1e-10 * np.abs(ref).max())
    check_counts(c, native)
    assert native.lane_counters == host.lane_counters


@pytest.mark.parametrize("wire", ["staged", "cores"])
def test_wire_formats(wire, monkeypatch):
    """Both ring wire formats (payload cores + halo rebuild, or whole staged
    payloads) give the oracle's tensor, through native rounds."""
    monkeypatch.setenv("G4RING_WIRE", wire)
    c = cfg(world_size=3, subring_size=3, lanes=2, measurements=8, batch=2, instrument=False, n_k=4, n_w=24,
            planes=30)
    rep = E.run_experiment(c)
    assert np.array_equal(rep.tensor, oracle_of(c))
    check_counts(c, rep)


def test_verify_harness_like_reference():
    """accuracy.verify (accuracy.py:108-128): float-mode ring runs pass the
    5e-7 gate for every seed; the corrupt negative control fails it."""
    from paper_2105_00027_b200 import accuracy as A
    c = cfg(world_size=2, subring_size=2, lanes=2, measurements=3, value_mode="float", n_k=4, n_w=8)
    res = A.verify(c, runs=2)
    assert res.passed and len(res.reports) == 2 and res.mean("l2_real") < 1e-12
    assert not A.verify(c, runs=1, corrupt=True).passed


@pytest.mark.parametrize("kw", [
    dict(value_mode="integer"),
    dict(value_mode="float"),
    dict(value_mode="float", dtype="c128g64"),
    dict(value_mode="float", dtype="c64"),
    dict(value_mode="integer", world_size=4, subring_size=2),               # 2 sub-rings + reduce
    dict(value_mode="float", direction="alternate", lanes=2),
])
def test_fused_ring_multi_plane_share(kw):
    """The ring in G4_ARITH_FUSED (the bench's arithmetic) with >= 16 planes per
    rank and >= 4 payloads per K1 pass, so every pass runs the deferred
    multi-plane kernel.  Integer payloads bitwise; float within 1e-12
    (c128), 1e-6 L1/L2 (c64-rounded payloads) and 1e-5 (c64 slices)."""
    base = dict(n_k=4, n_w=16, world_size=2, subring_size=2, lanes=1, measurements=8, batch=4, planes=64,
                arith="fused", instrument=False, seed=21)
    base.update(kw)
    c = cfg(**base)
    rep = E.run_experiment(c)
    ref = oracle_of(c)
    got = rep.tensor.astype(np.complex128)
    if c.value_mode == "integer":
        assert np.array_equal(got, ref)
    elif c.dtype == "c128":
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
    else:
        r = O.compare(ref, got)
        assert max(r["l1_real"], r["l1_imag"], r["l2_real"], r["l2_imag"]) < (1e-6 if c.dtype == "c128g64"
                                                                                 else 1e-5)
    for rr in range(c.world_size):
        assert rep.meas_counts[rr] == c.subring_size * c.measurements * c.lanes


def test_nccl_cross_subring_reduce():
    """north_star item 4: the final cross-sub-ring reduce as ncclReduce (one GPU
    per rank; skipped on a one-GPU box, where NCCL rejects ranks sharing a
    device): integer payloads sum exactly in any order."""
    import torch
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs (one per rank)")
    c = cfg(world_size=4, subring_size=2, lanes=2, measurements=3, reduce="nccl")
    rep = E.run_experiment(c)
    assert np.array_equal(rep.tensor, oracle_of(c))
