"""Host simulator of the ring schedule (TEST INFRASTRUCTURE).

Executes the per-rank operation lists of paper_2105_00027_b200.schedule with one
thread per (rank, stream), numpy payload buffers that carry their origin tuple
(like the reference wire header, wire.py:17-33), monotonic flags with
condition variables, CUDA-style events, and the CPU oracle as the accumulator.
It checks the host logic of the B200 ring (deadlock freedom, message laws,
exactly-once accumulation, lane isolation, final tensor) without a GPU.
"""
from __future__ import annotations

import threading

import numpy as np

from oracle import oracle as O
from paper_2105_00027_b200 import schedule as S


class SimDeadlock(Exception):
    def __init__(self, msg, rank, channel, value):
        super().__init__(msg)
        self.rank, self.channel, self.value = rank, channel, value


class RankState:
    def __init__(self, topo, pos, world_rank, subring, n, lo, hi, batch, channels):
        self.topo, self.pos, self.world_rank, self.subring = topo, pos, world_rank, subring
        self.channels = channels
        self.batch = batch
        self.flags = {(c.index, f): 0 for c in channels for f in (S.DATA, S.ACK_ACC, S.ACK_FWD)}
        self.cv = threading.Condition()
        self.bufs = {(c.index, b): [] for c in channels for b in (S.GEN, S.R0, S.R1)}
        self.g4 = np.zeros((hi - lo, n, n), np.complex128)
        self.lo, self.hi, self.n = lo, hi, n
        self.origins = {t: [] for t in range(topo.lanes)}
        self.sent = {t: 0 for t in range(topo.lanes)}
        self.received = {t: 0 for t in range(topo.lanes)}
        self.accumulated = {t: 0 for t in range(topo.lanes)}
        self.isolation_violations = 0
        self.events = {}
        self.ev_cv = threading.Condition()


def run_subring(topo, subring, n, lo_hi, seed, rounds, batch, mode="integer", steps=None,
                fault_rank=None, timeout=10.0, per_lane=False):
    """Run one sub-ring; returns the RankState list (index = position)."""
    s = topo.subring_size
    ranks = []
    for pos in range(s):
        lo, hi = lo_hi[pos]
        ranks.append(RankState(topo, pos, subring * s + pos, subring, n, lo, hi, batch,
                               S.make_channels(topo, pos, per_lane)))
    errors = []
    threads = []
    for st in ranks:
        ops = []
        for m in range(rounds):
            ops += S.round_schedule(topo, st.pos, st.channels, m, steps,
                                    skip_send_step0=(fault_rank == st.world_rank and m == 0))
        # bind every wait_event to the latest preceding record of that name
        seq = {}
        bound = []
        for op in ops:
            if op[0] == "record":
                seq[op[2]] = seq.get(op[2], 0) + 1
                bound.append(op + (seq[op[2]],))
            elif op[0] == "wait_event":
                bound.append(op + (seq.get(op[2], 0),))
            else:
                bound.append(op)
        streams = {}
        for op in bound:
            streams.setdefault(S.COMPUTE if op[0] in ("gen", "acc", "halo") else op[1], []).append(op)
        for name, lst in streams.items():
            th = threading.Thread(target=_stream_main, args=(ranks, st, lst, seed, mode, timeout, errors),
                                  daemon=True)
            threads.append(th)
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout * 4)
    if errors:
        raise errors[0]
    return ranks


def _stream_main(ranks, st, ops, seed, mode, timeout, errors):
    try:
        for op in ops:
            _execute(ranks, st, op, seed, mode, timeout)
    except Exception as exc:  # surfaced by run_subring
        errors.append(exc)
        with st.cv:
            st.cv.notify_all()


def _execute(ranks, st, op, seed, mode, timeout):
    kind = op[0]
    if kind == "gen":
        m = op[1]
        for c in st.channels:
            payloads = []
            for t in c.lanes:
                for b in range(st.batch):
                    meas = m * st.batch + b
                    up, down = O.gsigma(seed, st.world_rank, t, meas, st.n, mode)
                    payloads.append({"origin": (st.subring, st.pos, t, meas, st.world_rank),
                                     "up": up, "down": down})
            st.bufs[(c.index, S.GEN)] = payloads
    elif kind == "acc":
        for ci, buf in op[1]:
            c = st.channels[ci]
            for p in st.bufs[(ci, buf)]:
                O.accumulate(st.g4, st.lo, st.hi, p["up"], p["down"])
                lane = p["origin"][2]
                if lane not in c.lanes:
                    st.isolation_violations += 1
                st.origins[lane].append(p["origin"])
                st.accumulated[lane] += 1
                if buf != S.GEN:
                    st.received[lane] += 1
    elif kind == "wait":
        _, _, ci, flag, value = op
        with st.cv:
            if not st.cv.wait_for(lambda: st.flags[(ci, flag)] >= value, timeout):
                raise SimDeadlock(f"rank {st.world_rank} channel {ci} stalled waiting flag {flag} >= {value}",
                                  st.world_rank, ci, value)
    elif kind == "write":
        _, _, peer, ci, flag, value = op
        tgt = ranks[peer]
        with tgt.cv:
            tgt.flags[(ci_peer(tgt, st, ci), flag)] = max(tgt.flags[(ci_peer(tgt, st, ci), flag)], value)
            tgt.cv.notify_all()
    elif kind == "copy":
        _, _, ci, src, peer, dst = op
        tgt = ranks[peer]
        payloads = [dict(p, up=p["up"].copy(), down=p["down"].copy()) for p in st.bufs[(ci, src)]]
        tgt.bufs[(ci_peer(tgt, st, ci), dst)] = payloads
        for p in payloads:  # payloads (measurements) sent, per lane
            st.sent[p["origin"][2]] += 1
    elif kind == "halo":
        pass  # the simulator's payloads carry no halo
    elif kind == "record":
        with st.ev_cv:
            st.events[op[2]] = op[3]
            st.ev_cv.notify_all()
    elif kind == "wait_event":
        want = op[3]
        with st.ev_cv:
            if not st.ev_cv.wait_for(lambda: st.events.get(op[2], 0) >= want, timeout):
                raise SimDeadlock(f"rank {st.world_rank} event {op[2]} never recorded", st.world_rank, -1, want)
    else:  # pragma: no cover
        raise AssertionError(kind)


def ci_peer(tgt, src, ci):
    """The neighbour's channel index for the same lane group (same lanes -> same index)."""
    lanes = src.channels[ci].lanes
    for c in tgt.channels:
        if c.lanes == lanes:
            return c.index
    raise AssertionError("lane groups differ between neighbours")
