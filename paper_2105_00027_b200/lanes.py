"""The reference's per-lane ring driver over an injected communicator --
``LaneState``, ``run_measurement`` and ``rank_main(rt, world, cfg)`` of
ringacc/engine.py:96-161, 241-297, with the payloads and the G4 slice on the
GPU (K3 generates, K1 accumulates) and the transfers made by the caller's
communicator.

This is the drop-in path for a caller that owns its transport: any object with
the reference ``Communicator`` surface (transport/base.py:53-149: ``rank``,
``size``, ``isend(dest, tag, bytes)``, ``irecv(src, tag)`` returning an op
with ``wait()``, ``split(color, key)``, ``reduce_sum(ndarray, root)``) and a
runtime with ``spawn/join/now/make_lock``.  Payload bytes are the reference
wire format (wire.py), so ranks of this package and reference ranks
interoperate.  Each payload crosses the host twice per step, so this path is
transport-bound; the production path is ``engine.RingEngine`` (peer memory,
no host in the loop), which ``engine.rank_main(cfg)`` / ``run_experiment``
use.
"""
from __future__ import annotations

import json
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import schedule as S
from . import wire
from .errors import ContractViolation, DeadlockError
from .tensor import (CombinedIndexSpace, GSigma, GtSlice, Origin, accumulate_g4, fill_gsigma,
                     make_partition)

TAG_GATHER = 1 << 20          # engine.py:35-36
TAG_BLOB = (1 << 20) + 1


@dataclass
class LaneState:
    """One lane's three payload-sized device buffers, exchanged by handle swap
    only (engine.py:96-116)."""

    lane: int
    gsigma: GSigma
    send: GSigma
    recv: GSigma
    alloc_count: int = 0
    ring_phase_allocs: int = 0
    isolation_violations: int = 0
    origins_accumulated: list = field(default_factory=list)

    @classmethod
    def create(cls, space: CombinedIndexSpace, lane: int, tracker=None, rank: int = 0, *, device=None,
               dtype=torch.complex128) -> "LaneState":
        bufs = []
        for _ in range(3):
            g = GSigma.empty(space, device=device, dtype=dtype)
            if tracker is not None:
                tracker.alloc(rank, g.nbytes)
            bufs.append(g)
        return cls(lane, bufs[0], bufs[1], bufs[2], alloc_count=3)


class LaneRecorder:
    """Single-writer recorder of one lane's counters (instrument.py:36-67)."""

    enabled = True

    def __init__(self, counters, clock):
        self.counters = counters
        self._clock = clock

    def sent(self, nbytes: int) -> None:
        self.counters.envelopes_sent += 1
        self.counters.bytes_sent += nbytes
        self.counters.messages_sent += 1

    def received(self, nbytes: int) -> None:
        self.counters.envelopes_received += 1
        self.counters.bytes_received += nbytes

    def accumulated(self, seconds: float) -> None:
        self.counters.accumulations_applied += 1
        self.counters.accumulate_s += seconds

    def waited(self, seconds: float) -> None:
        self.counters.wait_s += seconds

    def now(self) -> float:
        return self._clock()

    def finish(self, started: float) -> None:
        self.counters.total_s = self._clock() - started


class NullRecorder:
    """Disabled instrumentation (instrument.py:70-96)."""

    enabled = False
    counters = None

    def sent(self, nbytes):
        pass

    def received(self, nbytes):
        pass

    def accumulated(self, seconds):
        pass

    def waited(self, seconds):
        pass

    def now(self):
        return 0.0

    def finish(self, started):
        pass


def run_measurement(topo, lane: LaneState, slice_: GtSlice, comm, lock, rec, seed: int, meas_index: int,
                    mode: str, subring_id: int, world_rank: int, rt=None, ring_steps: int | None = None,
                    fault: str | None = None) -> None:
    """One measurement of the pipeline ring for one lane (engine.py:119-161):
    K3 fills the lane's payload and K1 applies it; then for S-1 steps the
    payload goes right and the left neighbour's arrives through `comm`, and
    K1 applies each arrival.  Same step order, tags, counters, fault hook and
    DeadlockError diagnostic as the reference."""
    s = topo.subring_size
    origin = Origin(subring_id, comm.rank, lane.lane, meas_index, world_rank)
    fill_gsigma(lane.gsigma, seed, origin, mode)
    _accumulate(slice_, lane.gsigma, lock, rec, lane)
    lane.gsigma, lane.send = lane.send, lane.gsigma

    ring = S.lane_ring_id(topo, comm.rank, lane.lane)
    steps = s - 1 if ring_steps is None else ring_steps
    allocs_at_ring_start = lane.alloc_count
    for j in range(steps):
        if rt is not None and hasattr(rt, "annotate"):
            rt.annotate(rank=world_rank, lane=lane.lane, meas=meas_index, step=j)
        recv_op = comm.irecv(ring.recv_from, ring.tag)
        skip_send = fault == "skip-send" and j == 0
        if not skip_send:
            payload = wire.serialize_gsigma(lane.send)
            send_op = comm.isend(ring.send_to, ring.tag, payload)
            rec.sent(len(payload))
        t0 = rec.now()
        try:
            data = recv_op.wait()
        except Exception as exc:  # the communicator's own DeadlockError (any hierarchy)
            if not (isinstance(exc, DeadlockError) or type(exc).__name__ == "DeadlockError"):
                raise
            raise DeadlockError(f"rank {world_rank} lane {lane.lane} stalled at measurement "
                                f"{meas_index} step {j}: {exc}", rank=world_rank, lane=lane.lane,
                                step=j) from None
        rec.waited(rec.now() - t0)
        rec.received(len(data))
        wire.deserialize_gsigma_into(lane.recv, data)
        if lane.recv.origin.lane != lane.lane:
            lane.isolation_violations += 1
        _accumulate(slice_, lane.recv, lock, rec, lane)
        if not skip_send:
            t0 = rec.now()
            send_op.wait()
            rec.waited(rec.now() - t0)
        lane.send, lane.recv = lane.recv, lane.send
    lane.ring_phase_allocs += lane.alloc_count - allocs_at_ring_start


def _accumulate(slice_: GtSlice, g: GSigma, lock, rec, lane: LaneState) -> None:
    t0 = rec.now()
    with lock:
        accumulate_g4(slice_, g)
        if rec.enabled:  # the timer covers the device work, as the reference's covers numpy's
            torch.cuda.current_stream(slice_.data.device).synchronize()
    rec.accumulated(rec.now() - t0)
    if rec.enabled:
        o = g.origin
        lane.origins_accumulated.append((o.subring, o.rank, o.lane, o.meas, o.world_rank))


def _lane_main(rt, comm, topo, lane, rec, slice_, lock, cfg, world_rank, device) -> None:
    torch.cuda.set_device(device)  # runtime threads start on device 0
    started = rec.now()
    subring_id = world_rank // topo.subring_size
    fault_here = cfg.fault if (world_rank == 0 and lane.lane == 0) else None
    for m in range(cfg.measurements):
        run_measurement(topo, lane, slice_, comm, lock, rec, seed=cfg.seed, meas_index=m, mode=cfg.value_mode,
                        subring_id=subring_id, world_rank=world_rank, rt=rt,
                        ring_steps=cfg.ring_steps_override, fault=fault_here if m == 0 else None)
    torch.cuda.current_stream(device).synchronize()
    rec.finish(started)


def _device_for(world_rank: int) -> torch.device:
    return torch.device("cuda", world_rank % max(torch.cuda.device_count(), 1))


def comm_rank_main(rt, world, cfg):
    """rank_main(rt, world, cfg) over a reference-style communicator
    (engine.py:241-297): same sub-ring / position-group splits, partition,
    lane threads, canonical-order reduce and rank-0 report assembly."""
    from .engine import ExperimentReport, LaneCounters, RingTopology

    r = world.rank
    s = cfg.subring_size
    space = CombinedIndexSpace(cfg.n_k, cfg.n_w)
    topo = RingTopology(cfg.world_size, s, cfg.lanes, cfg.direction)
    t_start = rt.now()
    device = _device_for(r)
    torch.cuda.set_device(device)

    sub = world.split(r // s, r % s)
    pos = world.split(r % s, r // s)  # same-position group across sub-rings

    plan = make_partition(cfg.num_planes, s)
    lo, hi = plan.ranges[sub.rank]
    dtype = torch.complex64 if cfg.dtype == "c64" else torch.complex128
    pdtype = torch.complex128 if cfg.dtype == "c128" else torch.complex64
    slice_ = GtSlice.zeros(space, lo, hi, device=device, dtype=dtype)
    peak = slice_.nbytes

    lock = rt.make_lock() if hasattr(rt, "make_lock") else threading.Lock()
    lanes = [LaneState.create(space, t, None, r, device=device, dtype=pdtype) for t in range(cfg.lanes)]
    peak += sum(3 * ls.gsigma.device_nbytes for ls in lanes)
    recorders = [LaneRecorder(LaneCounters(), rt.now) if cfg.instrument else NullRecorder()
                 for _ in range(cfg.lanes)]
    handles = [rt.spawn(_lane_main, rt, sub, topo, lanes[t], recorders[t], slice_, lock, cfg, r, device,
                        name=(r, t)) for t in range(cfg.lanes)]
    rt.join(handles)
    torch.cuda.synchronize(device)

    reduced = pos.reduce_sum(slice_.data.to(torch.complex128).cpu().numpy(), root=0)

    blob = {
        "rank": r,
        "meas_count": slice_.meas_count,
        "slice": [lo, hi],
        "lanes": [{
            "lane": ls.lane,
            "counters": recorders[t].counters.to_dict() if cfg.instrument else None,
            "allocations": ls.alloc_count,
            "ring_phase_allocations": ls.ring_phase_allocs,
            "isolation_violations": ls.isolation_violations,
            "final_send_origin": [ls.send.origin.subring, ls.send.origin.rank, ls.send.origin.lane,
                                  ls.send.origin.meas, ls.send.origin.world_rank],
            "origins": ls.origins_accumulated,
        } for t, ls in enumerate(lanes)],
        "memory": {"peak": int(peak), "series": []},
    }
    world.isend(0, TAG_BLOB, json.dumps(blob).encode()).wait()
    if pos.rank == 0:
        world.isend(0, TAG_GATHER, wire.serialize_array(reduced)).wait()
    if r != 0:
        return None

    parts = [wire.deserialize_array(world.irecv(q, TAG_GATHER).wait()) for q in range(s)]
    full = np.concatenate(parts, axis=0)
    blobs = [json.loads(world.irecv(rr, TAG_BLOB).wait().decode()) for rr in range(world.size)]
    meas_counts, slices, peaks, counters, meta = {}, {}, {}, {}, {}
    for b in blobs:
        rr = b["rank"]
        meas_counts[rr] = b["meas_count"]
        slices[rr] = tuple(b["slice"])
        peaks[rr] = b["memory"]["peak"]
        for entry in b["lanes"]:
            key = (rr, entry["lane"])
            if entry["counters"] is not None:
                counters[key] = LaneCounters.from_dict(entry["counters"])
            meta[key] = {k: v for k, v in entry.items() if k != "counters"}
    return ExperimentReport(config=cfg.to_dict(), tensor=full, meas_counts=meas_counts, lane_counters=counters,
                            lane_meta=meta, memory_peaks=peaks, slices=slices,
                            elapsed_s=rt.now() - t_start, clock=getattr(rt, "clock_label", "monotonic"))
