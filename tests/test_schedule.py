"""Host logic of the B200 ring (CPU only): topology, channel grouping and the
per-rank operation schedule, executed by the host simulator (tests/ringsim.py)
against the oracle -- the reference's engine tests (tests/test_engine.py,
tests/test_acceptance.py C01/C03/C09/C10) restated for this engine."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2105_00027_b200 import schedule as S
from paper_2105_00027_b200.errors import ConfigError, ContractViolation

from . import ringsim


class TestTopology:
    def test_neighbors_wrap(self):
        topo = S.RingTopology(6, 3, 1)
        assert topo.left(0) == 2 and topo.right(0) == 1
        assert topo.left(2) == 1 and topo.right(2) == 0

    def test_validation(self):
        with pytest.raises(ConfigError):
            S.RingTopology(6, 4, 1)
        with pytest.raises(ConfigError):
            S.RingTopology(2, 2, 1000)
        with pytest.raises(ConfigError):
            S.RingTopology(2, 2, 1, "sideways")

    def test_lane_ring_ids(self):
        topo = S.RingTopology(3, 3, 2, "forward")
        for lane in (0, 1):
            ring = S.lane_ring_id(topo, 1, lane)
            assert (ring.recv_from, ring.send_to) == (0, 2) and ring.tag == 1000 + lane
        alt = S.RingTopology(3, 3, 2, "alternate")
        assert S.lane_ring_id(alt, 1, 0)[:2] == (0, 2)
        assert S.lane_ring_id(alt, 1, 1)[:2] == (2, 0)
        with pytest.raises(ContractViolation):
            S.lane_ring_id(alt, 0, 2)

    def test_channels_group_lanes_by_direction(self):
        assert [c.lanes for c in S.make_channels(S.RingTopology(4, 4, 3), 0)] == [(0, 1, 2)]
        ch = S.make_channels(S.RingTopology(4, 4, 5, "alternate"), 1)
        assert [c.lanes for c in ch] == [(0, 2, 4), (1, 3)]
        assert (ch[0].recv_from, ch[0].send_to) == (0, 2) and (ch[1].recv_from, ch[1].send_to) == (2, 0)

    def test_birth_position(self):
        # forward: the payload received at step j was born j+1 positions to the left
        assert [S.birth_position(0, j, 4, False) for j in range(3)] == [3, 2, 1]
        assert [S.birth_position(0, j, 4, True) for j in range(3)] == [1, 2, 3]


def run_world(world, s, lanes, rounds, batch, n, seed=1234, mode="integer", direction="forward",
              planes=None, steps=None, fault_rank=None, timeout=10.0, per_lane=False):
    topo = S.RingTopology(world, s, lanes, direction)
    planes = n if planes is None else planes
    ranges = O.partition(planes, s)
    subs = [ringsim.run_subring(topo, sub, n, ranges, seed, rounds, batch, mode, steps, fault_rank, timeout,
                                per_lane) for sub in range(world // s)]
    full = np.zeros((planes, n, n), np.complex128)
    for pos, (lo, hi) in enumerate(ranges):  # canonical rank-order reduce (base.py:135-148)
        total = subs[0][pos].g4.copy()
        for sub in subs[1:]:
            total += sub[pos].g4
        full[lo:hi] = total
    return topo, subs, full


def grid():
    for nk, nw in ((2, 2), (2, 3), (2, 4)):
        n = nk * nw
        for world in (2, 4, 6):
            if world > n:
                continue
            for s in range(1, world + 1):
                if world % s:
                    continue
                for lanes in (1, 3):
                    for rounds, batch in ((1, 1), (2, 2)):
                        yield n, world, s, lanes, rounds, batch


@pytest.mark.parametrize("n,world,s,lanes,rounds,batch", list(grid()))
def test_simulated_ring_equals_oracle(n, world, s, lanes, rounds, batch):
    """C01 + C03: bitwise oracle equality and the message laws on every grid point."""
    topo, subs, full = run_world(world, s, lanes, rounds, batch, n)
    m = rounds * batch
    ref = O.oracle_full(1234, n, world // s, s, lanes, m, "integer")
    assert np.array_equal(full, ref)
    for sub in subs:
        for st in sub:
            for t in range(lanes):
                assert st.sent[t] == (s - 1) * m
                assert st.received[t] == (s - 1) * m
                assert st.accumulated[t] == s * m
                # every origin of the sub-ring accumulated exactly once, lanes isolated
                assert len(st.origins[t]) == len(set(st.origins[t])) == s * m
                assert all(o[2] == t and o[0] == st.subring for o in st.origins[t])
            assert st.isolation_violations == 0


@pytest.mark.parametrize("world,s,lanes,direction", [(4, 4, 3, "forward"), (4, 2, 2, "forward"),
                                                     (6, 3, 3, "alternate"), (8, 4, 2, "forward")])
def test_lane_rings_equal_oracle(world, s, lanes, direction):
    """Every lane its own ring pipeline (lane_rings): same tensor, same laws."""
    n, rounds, batch = 8, 2, 2
    topo, subs, full = run_world(world, s, lanes, rounds, batch, n, direction=direction, per_lane=True)
    assert all(len(st.channels) == lanes for sub in subs for st in sub)
    m = rounds * batch
    assert np.array_equal(full, O.oracle_full(1234, n, world // s, s, lanes, m, "integer"))
    for sub in subs:
        for st in sub:
            for t in range(lanes):
                assert st.sent[t] == st.received[t] == (s - 1) * m and st.accumulated[t] == s * m
                assert len(st.origins[t]) == len(set(st.origins[t])) == s * m
            assert st.isolation_violations == 0


def test_lane_rings_template_periodic():
    topo = S.RingTopology(8, 4, 2, "forward")
    ch = S.make_channels(topo, 1, per_lane=True)
    assert [c.lanes for c in ch] == [(0,), (1,)] and [c.index for c in ch] == [0, 1]
    for par in (0, 1):
        tpl = S.steady_state_template(topo, 1, ch, par)
        assert len(tpl) == len(S.round_schedule(topo, 1, ch, 2 + par))


@pytest.mark.parametrize("direction", ["forward", "alternate"])
def test_direction_invariant(direction):
    _, _, a = run_world(4, 4, 3, 2, 1, 8, direction="forward")
    _, _, b = run_world(4, 4, 3, 2, 1, 8, direction=direction)
    assert np.array_equal(a, b)


def test_exchange_plane_subset():
    """north_star exchange planes: K3 in [0, P) with P < N, partitioned over S."""
    _, _, full = run_world(4, 4, 2, 2, 2, 12, planes=8)
    ref = O.oracle_full(1234, 12, 1, 4, 2, 4, "integer", 0, 8)
    assert np.array_equal(full, ref)


def test_matches_reference_engine_golden(golden):
    """Simulated B200 schedule vs the reference run_experiment outputs (engine.npz)."""
    e = golden("engine.npz")
    for i in range(4):
        nk, nw, world, s, lanes, m, seed = (int(x) for x in e[f"c{i}_cfg"])
        for mode in ("integer", "float"):
            _, _, full = run_world(world, s, lanes, m, 1, nk * nw, seed=seed, mode=mode)
            want = e[f"c{i}_{mode}_tensor"]
            if mode == "integer":
                assert np.array_equal(full, want)
            else:
                np.testing.assert_allclose(full, want, rtol=1e-12, atol=1e-12)
            ranges = O.partition(nk * nw, s)
            assert [tuple(r) for r in e[f"c{i}_{mode}_slices"]] == [ranges[r % s] for r in range(world)]


def test_short_ring_negative_control():
    topo, subs, full = run_world(3, 3, 1, 2, 1, 4, steps=1)
    for st in subs[0]:
        assert st.sent[0] == 1 * 2 and st.accumulated[0] == 2 * 2
    assert not np.array_equal(full, O.oracle_full(1234, 4, 1, 3, 1, 2, "integer"))


def test_skipped_send_deadlocks_with_diagnostic():
    with pytest.raises(ringsim.SimDeadlock) as err:
        run_world(2, 2, 1, 1, 1, 4, fault_rank=0, timeout=0.5)
    assert err.value.rank == 1 and err.value.channel == 0


def test_payload_ends_left_of_birth_rank():
    """After a round every forward payload sits at the left neighbour of its birth rank."""
    topo = S.RingTopology(4, 4, 1)
    sub = ringsim.run_subring(topo, 0, 4, O.partition(4, 4), 7, 1, 1)
    for st in sub:
        k_last = S.transfer_index(0, 2, 4)
        last = st.bufs[(0, S.R0 + k_last % 2)]
        assert last[0]["origin"][1] == (st.pos + 1) % 4


@pytest.mark.parametrize("world,s,lanes,direction", [(2, 2, 1, "forward"), (4, 4, 2, "forward"),
                                                     (4, 2, 2, "forward"), (3, 3, 3, "alternate"),
                                                     (8, 8, 1, "forward"), (8, 4, 2, "alternate")])
def test_steady_state_template_reproduces_rounds(world, s, lanes, direction):
    """The native round program's template (period 2, flag values affine in m)
    reproduces round_schedule for every steady-state round."""
    topo = S.RingTopology(world, s, lanes, direction)
    for pos in range(s):
        ch = S.make_channels(topo, pos)
        for par in (0, 1):
            tpl = S.steady_state_template(topo, pos, ch, par)
            for m in range(S.STEADY_FROM_ROUND, 12):
                if m % 2 != par:
                    continue
                got = S.round_schedule(topo, pos, ch, m)
                assert len(got) == len(tpl)
                for t, r in zip(tpl, got):
                    assert t[0] == r[0]
                    if t[0] in ("wait", "write"):
                        assert t[:-2] == r[:-1] and t[-2] + t[-1] * m == r[-1]
                    elif t[0] == "acc":
                        assert t == r[:2]
                    elif t[0] != "gen":
                        assert t == r
