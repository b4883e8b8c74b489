"""Drop-in replay of the reference engine tests (ringacc tests/test_engine.py:
83-235) against this package, through both of its ring drivers:

* the device ring -- ``engine.run_experiment(cfg)`` (one process per rank,
  payloads over peer memory);
* the communicator path -- ``engine.rank_main(rt, world, cfg)``, the reference
  signature, with a reference-style in-process communicator (tests/commsim.py)
  moving reference-wire-format payloads between rank threads.

Configs are the reference tests' ``desk_config`` overrides; each is checked
against every law those tests assert (oracle equality, counter conservation,
exactly-once origins, lane isolation, buffer conservation, payload position,
partition, JSON round trip) plus the negative controls.  GPU only.
"""
from dataclasses import replace

import numpy as np
import pytest

from oracle import oracle as O
from paper_2105_00027_b200 import engine as E
from paper_2105_00027_b200 import tensor as T
from paper_2105_00027_b200.errors import DeadlockError

from . import commsim

pytestmark = pytest.mark.gpu


def desk_config(**overrides):
    """The reference conftest's desk config (tests/conftest.py:6-12)."""
    base = dict(n_k=2, n_w=2, world_size=4, subring_size=2, lanes=1, measurements=2, seed=11,
                value_mode="integer", transport="inprocess", timeout_s=10.0)
    base.update(overrides)
    return E.ExperimentConfig(**base)


def oracle_of(c):
    return O.oracle_full(c.seed, c.space_size, c.world_size // c.subring_size, c.subring_size, c.lanes,
                         c.measurements, c.value_mode, 0, c.num_planes)


def run_comm(c):
    return commsim.run_world(c, E.rank_main, timeout_s=c.timeout_s)


def run_device(c):
    return E.run_experiment(c)


RUNNERS = {"comm": run_comm, "device": run_device}

# (test name in ringacc tests/test_engine.py, desk_config overrides)
CASES = [
    ("test_s1_degenerates_to_serial", dict(world_size=1, subring_size=1, lanes=1, measurements=1)),
    ("test_s3_message_and_accumulation_counts", dict(n_k=2, n_w=2, world_size=3, subring_size=3, measurements=4)),
    ("test_s4_bitwise_oracle_equality", dict(world_size=4, subring_size=4, lanes=2, measurements=3)),
    ("test_multiple_subrings_reduce", dict(n_k=2, n_w=3, world_size=6, subring_size=2, measurements=2)),
    ("test_exactly_once_per_origin", dict(world_size=4, subring_size=2, lanes=2, measurements=3)),
    ("test_lane_isolation", dict(world_size=4, subring_size=4, lanes=3, measurements=2)),
    ("test_payload_ends_left_of_birth_rank", dict(world_size=4, subring_size=4, lanes=1, measurements=2)),
    ("test_seven_lane_accumulation_count", dict(n_k=2, n_w=3, world_size=6, subring_size=3, lanes=7)),
    ("test_message_conservation", dict(n_k=2, n_w=3, world_size=6, subring_size=3, lanes=2)),
]
DEVICE_CASES = {"test_s4_bitwise_oracle_equality", "test_multiple_subrings_reduce",
                "test_seven_lane_accumulation_count", "test_payload_ends_left_of_birth_rank"}


def check_laws(c, rep):
    s, k, m, w = c.subring_size, c.lanes, c.measurements, c.world_size
    assert np.array_equal(rep.tensor, oracle_of(c))
    plan = T.make_partition(c.space_size, s)
    assert rep.slices == {r: plan.ranges[r % s] for r in range(w)}
    g = rep.registry().snapshot("global")
    assert g.envelopes_sent == g.envelopes_received == w * k * m * (s - 1)
    for r in range(w):
        c_r = rep.registry().snapshot("rank", rank=r)
        assert c_r.envelopes_sent == (s - 1) * m * k
        assert c_r.accumulations_applied == s * m * k
        assert rep.meas_counts[r] == s * m * k
        seen = []
        for t in range(k):
            meta = rep.lane_meta[(r, t)]
            assert meta["allocations"] == 3 and meta["ring_phase_allocations"] == 0
            assert meta["isolation_violations"] == 0
            origins = [tuple(o) for o in meta["origins"]]
            assert all(o[2] == t and o[0] == r // s for o in origins)
            seen += origins
            backward = c.direction == "alternate" and t % 2 == 1
            fso = meta["final_send_origin"]
            want = (r % s - 1) % s if backward else (r % s + 1) % s
            assert fso[1] == (want if s > 1 else r % s) and fso[2] == t and fso[3] == m - 1
        assert len(seen) == len(set(seen)) == s * m * k
    back = E.ExperimentReport.from_json_dict(rep.to_json_dict(), rep.tensor)
    assert back.meas_counts == rep.meas_counts and back.lane_counters == rep.lane_counters
    assert back.lane_meta.keys() == rep.lane_meta.keys() and back.slices == rep.slices
    assert back.memory_peaks == rep.memory_peaks and back.clock == rep.clock


@pytest.mark.parametrize("name,kw", CASES, ids=[c[0] for c in CASES])
def test_reference_engine_case_comm(name, kw):
    check_laws(desk_config(**kw), run_comm(desk_config(**kw)))


@pytest.mark.parametrize("name,kw", [c for c in CASES if c[0] in DEVICE_CASES],
                         ids=[c[0] for c in CASES if c[0] in DEVICE_CASES])
def test_reference_engine_case_device(name, kw):
    check_laws(desk_config(**kw), run_device(desk_config(**kw)))


@pytest.mark.parametrize("path", ["comm", "device"])
def test_direction_policy_invariant(path):
    c = desk_config(n_k=2, n_w=2, world_size=4, subring_size=4, lanes=3, measurements=2)
    fwd = RUNNERS[path](c)
    alt = RUNNERS[path](replace(c, direction="alternate"))
    assert np.array_equal(fwd.tensor, alt.tensor)
    check_laws(replace(c, direction="alternate"), alt)


def test_equivalence_across_subring_sizes_comm():
    tensors = [run_comm(desk_config(n_k=2, n_w=3, world_size=6, subring_size=s, lanes=2, measurements=2)).tensor
               for s in (1, 2, 3, 6)]
    for t in tensors[1:]:
        assert np.array_equal(tensors[0], t)


@pytest.mark.parametrize("path", ["comm", "device"])
def test_short_ring_breaks_counts_and_tensor(path):
    c = desk_config(n_k=2, n_w=2, world_size=3, subring_size=3, lanes=1, measurements=2, ring_steps_override=1)
    rep = RUNNERS[path](c)
    assert rep.registry().snapshot("rank", rank=0).envelopes_sent == 1 * 2
    assert rep.meas_counts[0] == 2 * 2
    assert not np.array_equal(rep.tensor, oracle_of(c))


@pytest.mark.parametrize("path", ["comm", "device"])
def test_skipped_send_deadlocks_with_diagnostic(path):
    c = desk_config(world_size=2, subring_size=2, lanes=1, measurements=1, fault="skip-send",
                    timeout_s=0.5 if path == "comm" else 3.0)
    with pytest.raises(DeadlockError) as err:
        RUNNERS[path](c)
    msg = str(err.value)
    assert "rank 1" in msg and "lane 0" in msg and "step 0" in msg


def test_comm_path_float_mode_and_mixed_payloads():
    """Float mode (1e-10, K3 device sin/cos) and complex64 wire-widened payloads
    on the communicator path."""
    c = desk_config(n_k=4, n_w=8, world_size=4, subring_size=2, lanes=2, measurements=2, value_mode="float")
    rep = run_comm(c)
    ref = oracle_of(c)
    np.testing.assert_allclose(rep.tensor, ref, rtol=1e-10, atol=1e-10 * np.abs(ref).max())
    rep = run_comm(replace(c, value_mode="integer", dtype="c128g64"))
    assert np.array_equal(rep.tensor, oracle_of(replace(c, value_mode="integer")))


def test_run_measurement_signature_and_wire_bytes(cuda_dev):
    """run_measurement / LaneState with the reference argument list on a 1-rank
    sub-ring, and the wire bytes of a device payload equal the reference format
    (wire.py:16-34: <7IQ header, up then down as <c16) built from the oracle."""
    import struct
    import threading

    from paper_2105_00027_b200 import wire

    space = T.CombinedIndexSpace(2, 4)
    n = space.size
    topo = E.RingTopology(1, 1, 1)
    lane = E.LaneState.create(space, 0, None, 0, device=cuda_dev)
    sl = T.GtSlice.zeros_full(space, device=cuda_dev)
    hub = commsim.Hub(1)
    rec = E.LaneRecorder(E.LaneCounters(), commsim.Runtime().now)
    E.run_measurement(topo, lane, sl, hub.comm(0), threading.Lock(), rec, seed=5, meas_index=3, mode="integer",
                      subring_id=0, world_rank=0)
    up, down = O.gsigma(5, 0, 0, 3, n, "integer")
    ref = np.zeros((n, n, n), np.complex128)
    O.accumulate(ref, 0, n, up, down)
    assert np.array_equal(sl.data.cpu().numpy(), ref) and sl.meas_count == 1
    assert rec.counters.accumulations_applied == 1 and lane.send.origin == T.Origin(0, 0, 0, 3, 0)
    blob = wire.serialize_gsigma(lane.send)
    want = struct.pack("<7IQ", 2, 4, 0, 0, 0, 3, 0, 2 * n * n * 16) + up.astype("<c16").tobytes() + \
        down.astype("<c16").tobytes()
    assert blob == want
    g = T.GSigma.empty(space, device=cuda_dev)
    wire.deserialize_gsigma_into(g, want)
    assert np.array_equal(g.up.cpu().numpy(), up) and np.array_equal(g.down.cpu().numpy(), down)
    assert g.origin == T.Origin(0, 0, 0, 3, 0)
