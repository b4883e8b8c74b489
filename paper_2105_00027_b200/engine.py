"""Ring driver on B200s -- the replacement of ``ringacc.engine``
(/root/reference/pkg/src/ringacc/engine.py) for device-resident payloads.

One process per GPU.  ``torch.distributed`` (gloo) is the control plane only:
rendezvous, communicator splits, the one-time exchange of CUDA IPC handles,
barriers.  The data path never touches the host:

* payload transfers are copy-engine peer copies of the payload cores
  (``g4_copy_payload_cores``) straight into the right neighbour's receive slot
  over NVLink/NVSwitch (no SM cycles); the receiver rebuilds the staged halo
  (``g4_fill_halo``) before its K1 pass;
* ordering is carried by 64-bit sequence flags in the receiver's / sender's
  memory, written with ``cuStreamWriteValue64`` and awaited with
  ``cuStreamWaitValue64`` (``g4_flag_write`` / ``g4_flag_wait``): no host round
  trip per step, and the K1 pass over the payload received at step j runs on
  the compute stream while the comm stream forwards that same payload (and
  receives the next one);
* the schedule of every round is the host-logic plan of ``schedule.py``; from
  round 2 on a round is one native call (``g4_round_program_run``);
* the end-of-run cross-sub-ring reduction sums matching slices in canonical
  rank order with a kernel that reads the peers' slices over NVLink
  (``g4_reduce_sum``), bitwise equal to the reference's ``reduce_sum``.

Several ranks may share one GPU (the same code path; peer copies become local
copies), which is how the multi-rank path is tested on a single B200.
"""
from __future__ import annotations

import ctypes
import json
import os
import socket
import time
from dataclasses import asdict, dataclass, field, fields

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from . import schedule as S
from .errors import ConfigError, ContractViolation, DeadlockError
from .schedule import LaneRing, RingTopology, lane_ring_id  # noqa: F401  (re-exported API)
from .tensor import (CombinedIndexSpace, GtSlice, Origin, _dtype_code, accumulate_dtype_code,
                     make_partition, staged_shape)

VALUE_MODES = ("float", "integer")
ARITH_MODES = {"exact": _lib.G4_ARITH_EXACT, "fused": _lib.G4_ARITH_FUSED}
_MODE_CODE = {"float": _lib.G4_MODE_FLOAT, "integer": _lib.G4_MODE_INTEGER}


@dataclass
class ExperimentConfig:
    """Run shape -- every field of ringacc.config.ExperimentConfig
    (config.py:46-66, same names, order and defaults, so reference keyword and
    positional constructions both work), plus the B200 extensions (keyword
    only in practice; they follow the reference fields).

    ``transport``, ``link``, ``out_dir``, ``sweep`` and ``memory`` are accepted
    and validated like the reference but do not steer the device ring: its
    payloads always move over peer memory (NVLink), and the sweep/memory
    settings belong to the reference's CLI models (model.py holds those).
    ``transport`` selects the data path only on the communicator path
    (``rank_main(rt, world, cfg)`` with a reference-style communicator)."""

    n_k: int
    n_w: int
    world_size: int
    subring_size: int
    lanes: int
    measurements: int
    seed: int = 0
    value_mode: str = "float"
    transport: str = "inprocess"
    direction: str = "forward"
    link: object = None
    timeout_s: float = 30.0
    instrument: bool = True
    out_dir: str | None = None
    sweep: object = None
    memory: object = None
    # B200 extensions
    planes: int | None = None      # exchange planes K3 in [0, planes); None = all N (reference)
    batch: int = 1                 # measurements per lane carried by one ring message / K1 pass
    dtype: str = "c128"            # "c128" (reference), "c64", or "c128g64" (c128 G4, c64 payloads)
    gather: bool = True            # assemble the full tensor on world rank 0
    sample_planes: tuple[int, ...] = ()  # K3 planes copied to world rank 0 (report.samples)
    arith: str = "exact"           # K1 arithmetic: "exact" (bitwise reference order) or "fused" (FMA
                                   # chains + deferred update, within 1e-12; g4_set_arith_mode)
    reduce: str = "peer"           # cross-sub-ring reduce: "peer" (one kernel reading the peers' slices
                                   # over NVLink, canonical rank order, bitwise = reference) or "nccl"
                                   # (ncclReduce of the slices viewed as float64; needs one GPU per rank)
    lane_rings: bool = False       # every lane its own ring pipeline (comm stream, flags, buffers),
                                   # as the reference's per-lane rings; False: lanes sharing a
                                   # direction share one channel (one copy per step)
    # test hooks (never part of a user config, as in the reference)
    ring_steps_override: int | None = None
    fault: str | None = None

    @property
    def space_size(self) -> int:
        return self.n_k * self.n_w

    @property
    def num_planes(self) -> int:
        return self.space_size if self.planes is None else self.planes

    def to_dict(self) -> dict:
        return asdict(self)


TRANSPORTS = ("inprocess", "sim", "tcp")


def as_config(cfg) -> ExperimentConfig:
    """This package's config from a reference ``ringacc.config.ExperimentConfig``
    (or any object with its attributes, or a dict of its fields).  Fields the
    reference does not have keep their defaults."""
    if isinstance(cfg, ExperimentConfig):
        return cfg
    names = [f.name for f in fields(ExperimentConfig)]
    if isinstance(cfg, dict):
        unknown = sorted(set(cfg) - set(names))
        if unknown:
            raise ConfigError(f"unknown config key(s): {', '.join(unknown)}")
        return ExperimentConfig(**cfg)
    kw = {k: getattr(cfg, k) for k in names if hasattr(cfg, k)}
    missing = [k for k in ("n_k", "n_w", "world_size", "subring_size", "lanes", "measurements") if k not in kw]
    if missing:
        raise ConfigError(f"missing required config key: {missing[0]}")
    return ExperimentConfig(**kw)


def validate_config(cfg) -> None:
    """config.py:156-185 semantics (ConfigError), plus the extensions.  Accepts
    a reference config too (as_config)."""
    cfg = as_config(cfg)
    for name in ("n_k", "n_w", "world_size", "subring_size", "lanes", "measurements", "batch"):
        v = getattr(cfg, name)
        if not isinstance(v, int) or v < 1:
            raise ConfigError(f"{name} must be an integer >= 1, got {v!r}")
    if not isinstance(cfg.seed, int) or cfg.seed < 0:
        raise ConfigError(f"seed must be a non-negative integer, got {cfg.seed!r}")
    if cfg.world_size % cfg.subring_size != 0:
        raise ConfigError(f"subring_size {cfg.subring_size} does not divide world_size {cfg.world_size}")
    if cfg.planes is None and cfg.world_size > cfg.space_size:
        raise ConfigError(f"world_size {cfg.world_size} exceeds combined index count {cfg.space_size}: "
                          "some rank would own an empty slice")
    if not (1 <= cfg.num_planes <= cfg.space_size):
        raise ConfigError(f"planes must be in [1, {cfg.space_size}], got {cfg.num_planes}")
    if cfg.subring_size > cfg.num_planes:
        raise ConfigError(f"subring_size {cfg.subring_size} exceeds the {cfg.num_planes} exchange planes: "
                          "some rank would own an empty slice")
    if cfg.lanes >= S.MAX_LANES:
        raise ConfigError(f"lanes must be < {S.MAX_LANES} (tag stride), got {cfg.lanes}")
    if cfg.value_mode not in VALUE_MODES:
        raise ConfigError(f"value_mode must be one of {VALUE_MODES}, got {cfg.value_mode!r}")
    if cfg.transport not in TRANSPORTS:
        raise ConfigError(f"transport must be one of {TRANSPORTS}, got {cfg.transport!r}")
    if cfg.direction not in ("forward", "alternate"):
        raise ConfigError(f"direction must be forward or alternate, got {cfg.direction!r}")
    if cfg.dtype not in ("c128", "c64", "c128g64"):
        raise ConfigError(f"dtype must be c128, c64 or c128g64, got {cfg.dtype!r}")
    if cfg.timeout_s <= 0:
        raise ConfigError("timeout_s must be positive")
    if cfg.reduce not in ("peer", "nccl"):
        raise ConfigError(f"reduce must be peer or nccl, got {cfg.reduce!r}")
    if cfg.arith not in ARITH_MODES:
        raise ConfigError(f"arith must be one of {tuple(ARITH_MODES)}, got {cfg.arith!r}")


# ---------------------------------------------------------------------------
# control plane

class Control:
    """A group of ranks for control messages (torch.distributed, gloo)."""

    def __init__(self, group=None, ranks: tuple[int, ...] | None = None):
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.world_ranks = ranks if ranks is not None else tuple(range(dist.get_world_size()))
            self.rank = self.world_ranks.index(dist.get_rank())
        else:
            self.world_ranks = (0,)
            self.rank = 0
        self.size = len(self.world_ranks)

    def allgather(self, obj) -> list:
        if self.size == 1:
            return [obj]
        out = [None] * self.size
        dist.all_gather_object(out, obj, group=self.group)
        return out

    def barrier(self) -> None:
        if self.size > 1:
            dist.barrier(group=self.group)

    def split(self, color: int, key: int) -> "Control":
        """Communicator split (transport/base.py:92-124): groups by color, ranked
        by (key, parent rank).  Collective over all ranks of this group."""
        entries = self.allgather((color, key, self.rank))
        groups: dict[int, list[tuple[int, int]]] = {}
        for c, k, r in entries:
            groups.setdefault(c, []).append((k, r))
        mine = None
        for c in sorted(groups):
            members = tuple(self.world_ranks[r] for _, r in sorted(groups[c]))
            g = dist.new_group(list(members)) if self.size > 1 else None  # every rank creates every group
            if c == color:
                mine = (g, members)
        return Control(*mine)


def build_subrings(world: Control, subring_size: int) -> Control:
    """Consecutive ranks form each sub-ring: color r // S, key r % S (engine.py:86-92)."""
    if world.size % subring_size != 0:
        raise ConfigError(f"subring size {subring_size} does not divide world size {world.size}")
    return world.split(world.rank // subring_size, world.rank % subring_size)


# ---------------------------------------------------------------------------
# peer memory helpers

def export_ptr(ptr: int) -> tuple[bytes, int]:
    lib = _lib.load()
    h = ctypes.create_string_buffer(_lib.G4_IPC_HANDLE_BYTES)
    off = ctypes.c_int64()
    _lib.check(lib.g4_ipc_export(ptr, h, ctypes.byref(off)), "ipc_export")
    return h.raw, off.value


class PeerMap:
    """Imported peer pointers of this process (closed together)."""

    def __init__(self):
        self.ptrs: list[int] = []

    def open(self, handle: bytes, offset: int, local_ptr: int | None = None) -> int:
        if local_ptr is not None:  # our own buffer: no IPC needed
            return local_ptr
        lib = _lib.load()
        out = ctypes.c_void_p()
        _lib.check(lib.g4_ipc_import(handle, offset, ctypes.byref(out)), "ipc_import")
        self.ptrs.append(out.value)
        return out.value

    def close(self) -> None:
        lib = _lib.load()
        for p in self.ptrs:
            lib.g4_ipc_close(p)
        self.ptrs = []


def reduce_sum(ctl: Control, data: torch.Tensor, root: int = 0) -> None:
    """Entrywise sum of the members' `data` into root's `data`, in canonical rank
    order 0, 1, 2, ... (transport/base.py:126-149), reading peers' tensors over
    NVLink with one kernel.  Collective over `ctl`."""
    if ctl.size == 1:
        return
    dev = data.device
    torch.cuda.current_stream(dev).synchronize()
    me = (export_ptr(data.data_ptr()), tuple(data.shape), str(data.dtype))
    allm = ctl.allgather(me)
    if any(m[1:] != me[1:] for m in allm):
        raise ContractViolation("reduce_sum shape/dtype mismatch across ranks")
    if ctl.rank == root:
        pm = PeerMap()
        try:
            srcs = [pm.open(h, off, data.data_ptr() if r == ctl.rank else None)
                    for r, ((h, off), _, _) in enumerate(allm)]
            lib = _lib.load()
            stream = torch.cuda.current_stream(dev)
            _lib.check(lib.g4_reduce_sum(data.data_ptr(), _lib.ptr_array(srcs), len(srcs), data.numel(),
                                         _dtype_code(data.dtype), stream.cuda_stream), "reduce_sum")
            stream.synchronize()
        finally:
            pm.close()
    ctl.barrier()


_NCCL_GROUPS: dict[tuple[int, ...], object] = {}


def reduce_sum_nccl(world: Control, s: int, data: torch.Tensor) -> None:
    """The cross-sub-ring reduce as an NCCL collective (north_star item 4): the
    position group of this rank (world ranks r % S + S*i) sums its slices into
    the group's first member with ncclReduce, the complex slice viewed as
    float64 (an entrywise sum of real and imaginary parts).  NCCL picks the
    summation order, so float results agree with the canonical-order reference
    within rounding (integer-valued payloads stay exact); "peer" is the
    bitwise path.  Collective over the whole world (every rank creates every
    group's communicator)."""
    if world.size // s == 1:
        return
    if torch.cuda.device_count() < world.size:
        raise ConfigError("reduce='nccl' needs one GPU per rank (NCCL rejects ranks sharing a device)")
    mine = None
    for c in range(s):
        members = tuple(world.world_ranks[c + s * i] for i in range(world.size // s))
        g = _NCCL_GROUPS.get(members)
        if g is None:  # communicators are created once per member set and reused by later runs
            g = _NCCL_GROUPS[members] = dist.new_group(list(members), backend="nccl")
        if world.rank % s == c:
            mine = (g, members[0])
    torch.cuda.current_stream(data.device).synchronize()
    dist.reduce(torch.view_as_real(data), dst=mine[1], op=dist.ReduceOp.SUM, group=mine[0])
    torch.cuda.current_stream(data.device).synchronize()
    world.barrier()


# ---------------------------------------------------------------------------
# the per-rank ring executor

@dataclass
class LaneCounters:
    """Per-(rank, lane) counters: the fields of ringacc.instrument.CounterSet
    (instrument.py:14-33, same names and meaning) plus ``messages_sent`` (ring
    messages, one per step, each carrying `batch` payloads).  The device ring
    fills the counts; its timers stay 0 (device time is in round_ms)."""

    envelopes_sent: int = 0       # payloads (measurements) forwarded to the next rank
    envelopes_received: int = 0
    bytes_sent: int = 0
    bytes_received: int = 0
    accumulations_applied: int = 0
    wait_s: float = 0.0
    accumulate_s: float = 0.0
    total_s: float = 0.0
    messages_sent: int = 0

    def add(self, other) -> None:
        for f in fields(self):
            setattr(self, f.name, getattr(self, f.name) + getattr(other, f.name, 0))

    def to_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_dict(cls, d: dict) -> "LaneCounters":
        return cls(**{f.name: d.get(f.name, 0) for f in fields(cls)})


@dataclass
class CounterRegistry:
    """All lanes' counters of one experiment (instrument.py:103-131)."""

    clock_label: str = "cuda-event"
    lanes: dict = field(default_factory=dict)

    def register(self, rank: int, lane: int, counters) -> None:
        self.lanes[(rank, lane)] = counters

    def snapshot(self, scope: str = "global", rank: int | None = None, lane: int | None = None) -> LaneCounters:
        """Aggregate counters at lane, rank, or global scope."""
        out = LaneCounters()
        for (r, t), c in self.lanes.items():
            if scope == "lane" and (r, t) != (rank, lane):
                continue
            if scope == "rank" and r != rank:
                continue
            out.add(c)
        return out

    def per_rank(self) -> dict:
        ranks: dict[int, LaneCounters] = {}
        for (r, _), c in self.lanes.items():
            ranks.setdefault(r, LaneCounters()).add(c)
        return ranks


class RingEngine:
    """Everything one rank of one sub-ring does on its GPU."""

    def __init__(self, cfg: ExperimentConfig, sub: Control, world_rank: int, device: torch.device):
        self.cfg = cfg
        self.sub = sub
        self.world_rank = world_rank
        self.device = device
        self.pos = sub.rank
        self.subring = world_rank // cfg.subring_size
        self.topo = RingTopology(cfg.world_size, cfg.subring_size, cfg.lanes, cfg.direction)
        self.space = CombinedIndexSpace(cfg.n_k, cfg.n_w)
        n = self.space.size
        self.lo, self.hi = make_partition(cfg.num_planes, cfg.subring_size).ranges[self.pos]
        self.dtype = torch.complex64 if cfg.dtype == "c64" else torch.complex128         # G4 slice
        self.pdtype = torch.complex128 if cfg.dtype == "c128" else torch.complex64       # payloads
        self.code = accumulate_dtype_code(self.dtype, self.pdtype)
        self.pcode = _dtype_code(self.pdtype)
        self.slice = GtSlice.zeros(self.space, self.lo, self.hi, device=device, dtype=self.dtype)
        self.channels = S.make_channels(self.topo, self.pos, per_lane=cfg.lane_rings)
        self.lib = _lib.load()
        _lib.check(self.lib.g4_preload_ring_kernels(), "preload_ring_kernels")
        # per channel: 3 buffers (GEN, R0, R1) x batch x lanes staged payloads
        self.bufs = [torch.zeros((3, cfg.batch * len(c.lanes)) + staged_shape(n, self.pdtype), dtype=self.pdtype,
                                 device=device) for c in self.channels]
        self.payload_bytes = int(np.prod(staged_shape(n, self.pdtype))) * self.bufs[0].element_size()
        # wire format: payload cores (default) or whole staged payloads (G4RING_WIRE=staged,
        # for A/B on nodes where strided peer copies are slow; no halo rebuild then)
        self.wire_cores = os.environ.get("G4RING_WIRE", "cores") != "staged"
        self.wire_bytes = (2 * n * n * self.bufs[0].element_size() if self.wire_cores else self.payload_bytes)
        self.flags = torch.zeros(len(self.channels) * S.FLAGS_PER_CHANNEL, dtype=torch.int64, device=device)
        self.compute = torch.cuda.Stream(device)
        self.comm = [torch.cuda.Stream(device) for _ in self.channels]
        self.events: dict[str, torch.cuda.Event] = {}
        self.counters = {t: LaneCounters() for t in range(cfg.lanes)}
        self.origins = {t: [] for t in range(cfg.lanes)}
        self.meas_count = 0
        self.peers = PeerMap()
        self.kernel_events: list[tuple[torch.cuda.Event, torch.cuda.Event]] | None = None
        self.next_round = 0
        self._prog = [None, None]  # native round programs by round parity
        self._prog_delta = None
        self.native = self._native_ok()
        self._make_events()
        self._connect()

    # -- setup --------------------------------------------------------------
    def _connect(self) -> None:
        mine = {"flags": export_ptr(self.flags.data_ptr()),
                "bufs": [export_ptr(b.data_ptr()) for b in self.bufs],
                "lanes": [c.lanes for c in self.channels]}
        torch.cuda.synchronize(self.device)
        everyone = self.sub.allgather(mine)
        self.peer_flags: dict[int, int] = {}
        self.peer_bufs: dict[tuple[int, int], int] = {}
        for c in self.channels:
            for p in (c.send_to, c.recv_from):
                local = p == self.pos
                if p not in self.peer_flags:
                    h, off = everyone[p]["flags"]
                    self.peer_flags[p] = self.peers.open(h, off, self.flags.data_ptr() if local else None)
            if everyone[c.send_to]["lanes"][c.index] != c.lanes:
                raise ContractViolation("neighbouring ranks disagree on lane grouping")
            h, off = everyone[c.send_to]["bufs"][c.index]
            self.peer_bufs[(c.send_to, c.index)] = self.peers.open(
                h, off, self.bufs[c.index].data_ptr() if c.send_to == self.pos else None)

    def close(self) -> None:
        torch.cuda.synchronize(self.device)
        self.sub.barrier()
        for i, prog in enumerate(self._prog):
            if prog is not None:
                self.lib.g4_round_program_destroy(prog)
                self._prog[i] = None
        self.peers.close()

    # -- helpers --------------------------------------------------------------
    def _stream(self, name: str) -> torch.cuda.Stream:
        return self.compute if name == S.COMPUTE else self.comm[int(name[4:])]

    def _buf_ptr(self, ci: int, buf: int, i: int = 0) -> int:
        return self.bufs[ci][buf, i].data_ptr()

    def _nb(self, m: int) -> int:
        """Measurements per lane in round m (the last round may be partial)."""
        return min(self.cfg.batch, self.cfg.measurements - m * self.cfg.batch)

    def _flag_off(self, ci: int, flag: int) -> int:
        return (ci * S.FLAGS_PER_CHANNEL + flag) * 8

    # -- native round program ---------------------------------------------------
    def _native_ok(self) -> bool:
        """Rounds are issued by the native program (one C call per round) unless
        the run needs per-op host work: origin tracking, fault injection, a
        truncated ring, or a partial last round.  G4RING_NATIVE=0 forces the
        per-op host loop (A/B and parity tests)."""
        cfg = self.cfg
        return (os.environ.get("G4RING_NATIVE", "1") != "0" and not cfg.instrument and cfg.fault is None
                and cfg.ring_steps_override is None and cfg.measurements % cfg.batch == 0)

    NATIVE_FROM_ROUND = S.STEADY_FROM_ROUND

    def _program(self, m: int):
        """Compile the steady-state schedule of round parity m % 2
        (schedule.steady_state_template: flag values affine in the round
        number) into the native op list of g4_round_program_create.  Rounds 0
        and 1 run the host loop; stream events are shared with it."""
        par = m % 2
        if self._prog[par] is not None:
            return self._prog[par]
        cfg = self.cfg
        template = S.steady_state_template(self.topo, self.pos, self.channels, par)
        streams = [self.compute] + self.comm
        sidx = lambda name: 0 if name == S.COMPUTE else 1 + int(name[4:])  # noqa: E731
        ev_names = list(self.events)
        words, ptrs, meta = [], [], []
        lanes = range(cfg.lanes)
        delta = {"acc": dict.fromkeys(lanes, 0), "recv": dict.fromkeys(lanes, 0), "sent": dict.fromkeys(lanes, 0),
                 "msgs": dict.fromkeys(lanes, 0), "bytes": dict.fromkeys(lanes, 0), "meas": 0}
        nb = cfg.batch

        for op in template:
            kind = op[0]
            if kind == "gen":
                off, moff = len(ptrs), len(meta)
                wr, ln, mb = [], [], []
                for c in self.channels:
                    for b in range(nb):
                        for li, t in enumerate(c.lanes):
                            ptrs.append(self._buf_ptr(c.index, S.GEN, b * len(c.lanes) + li))
                            wr.append(self.world_rank)
                            ln.append(t)
                            mb.append(b)
                meta += wr + ln + mb
                words.append([_lib.G4_OP_GEN, 0, off, len(wr), moff, 0, 0, 0])
            elif kind == "acc":
                off = len(ptrs)
                for ci, buf in op[1]:
                    c = self.channels[ci]
                    ptrs += [self._buf_ptr(ci, buf, j) for j in range(nb * len(c.lanes))]
                    for t in c.lanes:
                        delta["acc"][t] += nb
                        if buf != S.GEN:
                            delta["recv"][t] += nb
                words.append([_lib.G4_OP_ACC, 0, off, len(ptrs) - off, 0, 0, 0, 0])
                delta["meas"] += len(ptrs) - off
            elif kind == "wait":
                _, st, ci, flag, base, slope = op
                words.append([_lib.G4_OP_WAIT, sidx(st), self.flags.data_ptr() + self._flag_off(ci, flag),
                              base, slope, 0, 0, 0])
            elif kind == "write":
                _, st, peer, ci, flag, base, slope = op
                words.append([_lib.G4_OP_WRITE, sidx(st), self.peer_flags[peer] + self._flag_off(ci, flag),
                              base, slope, 0, 0, 0])
            elif kind == "copy":
                _, st, ci, src, peer, dst = op
                c = self.channels[ci]
                cnt = nb * len(c.lanes)
                dst_ptr = self.peer_bufs[(peer, ci)] + dst * self.bufs[ci][0].numel() * self.bufs[ci].element_size()
                if self.wire_cores:
                    words.append([_lib.G4_OP_COPY, sidx(st), dst_ptr, self._buf_ptr(ci, src), 0, cnt,
                                  self.space.size, self.pcode])
                else:
                    words.append([_lib.G4_OP_COPY, sidx(st), dst_ptr, self._buf_ptr(ci, src),
                                  cnt * self.payload_bytes, 0, 0, 0])
                for t in c.lanes:
                    delta["sent"][t] += nb
                    delta["msgs"][t] += 1
                    delta["bytes"][t] += nb * self.wire_bytes
            elif kind == "halo":
                if not self.wire_cores:
                    continue
                off = len(ptrs)
                for ci, buf in op[1]:
                    ptrs += [self._buf_ptr(ci, buf, j) for j in range(nb * len(self.channels[ci].lanes))]
                words.append([_lib.G4_OP_HALO, 0, off, len(ptrs) - off, 0, 0, 0, 0])
            elif kind in ("record", "wait_event"):
                words.append([_lib.G4_OP_RECORD if kind == "record" else _lib.G4_OP_WAIT_EVENT,
                              sidx(op[1]), ev_names.index(op[2]), 0, 0, 0, 0, 0])
            else:  # pragma: no cover
                raise AssertionError(kind)
        flat = [w for op in words for w in op]
        prog = ctypes.c_void_p()
        _lib.check(self.lib.g4_round_program_create(
            _lib.i64_array(flat), len(words), _lib.ptr_array(ptrs), len(ptrs), _lib.i64_array(meta or [0]),
            len(meta), _lib.ptr_array([st.cuda_stream for st in streams]), len(streams),
            _lib.ptr_array([self.events[k].cuda_event for k in ev_names]), len(ev_names),
            self.slice.data.data_ptr(), self.lo, self.hi, self.space.size, self.code, self.pcode,
            cfg.seed & 0xFFFFFFFFFFFFFFFF, _MODE_CODE[cfg.value_mode], cfg.batch, 1, ctypes.byref(prog)),
            "round_program_create")
        self._prog[par], self._prog_delta = prog, delta
        return prog

    def _make_events(self) -> None:
        """Create every named stream event of the schedule up front (recorded
        once so the CUDA event exists), shared by host-loop and native rounds."""
        names = []
        for m in range(4):
            for op in S.round_schedule(self.topo, self.pos, self.channels, m):
                if op[0] in ("record", "wait_event") and op[2] not in names:
                    names.append(op[2])
        for name in names:
            ev = torch.cuda.Event()
            ev.record(self.compute)
            self.events[name] = ev
        self.compute.synchronize()

    def k1_mean_ms(self) -> float:
        """Mean K1 launch duration of the last completed round (native rounds),
        or over the launches recorded in kernel_events (host-loop rounds)."""
        last = (self.next_round - 1) % 2
        if self.native and self.next_round > self.NATIVE_FROM_ROUND and self._prog[last] is not None:
            mean, cnt = ctypes.c_double(), ctypes.c_int32()
            _lib.check(self.lib.g4_round_program_k1_ms(self._prog[last], ctypes.byref(mean), ctypes.byref(cnt)),
                       "round_program_k1_ms")
            return mean.value
        if not self.kernel_events:
            raise ContractViolation("no K1 launches were timed")
        return float(np.mean([a.elapsed_time(b) for a, b in self.kernel_events]))

    # -- one round ------------------------------------------------------------
    def enqueue_round(self, m: int | None = None, regenerate: bool = True) -> None:
        """Enqueue the next round (asynchronous).  Rounds must be consecutive:
        transfer indices (and therefore the flags) are derived from the round
        number.  `m` defaults to the next round; regenerate=False reuses the
        payloads already in GEN (benchmarking with resident inputs)."""
        if m is None:
            m = self.next_round
        if m != self.next_round:
            raise ContractViolation(f"rounds must be consecutive: expected {self.next_round}, got {m}")
        self.next_round = m + 1
        cfg = self.cfg
        if self.native and m >= self.NATIVE_FROM_ROUND:
            _lib.check(self.lib.g4_round_program_run(self._program(m), m, int(regenerate)), "round_program_run")
            d = self._prog_delta
            for t, cnt in self.counters.items():
                cnt.accumulations_applied += d["acc"][t]
                cnt.envelopes_received += d["recv"][t]
                cnt.bytes_received += d["recv"][t] * self.wire_bytes
                cnt.envelopes_sent += d["sent"][t]
                cnt.messages_sent += d["msgs"][t]
                cnt.bytes_sent += d["bytes"][t]
            self.slice.meas_count += d["meas"]
            self.meas_count += d["meas"]
            return
        nb = max(1, min(self._nb(m), cfg.batch)) if regenerate else cfg.batch
        fault = cfg.fault == "skip-send" and self.world_rank == 0 and m == 0
        ops = S.round_schedule(self.topo, self.pos, self.channels, m, cfg.ring_steps_override, fault)
        if not regenerate:
            ops = [op for op in ops if op[0] != "gen"]
        lib = self.lib
        s = cfg.subring_size
        for op in ops:
            kind = op[0]
            if kind == "gen":
                ptrs, wr, lanes, meas = [], [], [], []
                for c in self.channels:
                    for b in range(nb):
                        for li, t in enumerate(c.lanes):
                            ptrs.append(self._buf_ptr(c.index, S.GEN, b * len(c.lanes) + li))
                            wr.append(self.world_rank)
                            lanes.append(t)
                            meas.append(m * cfg.batch + b)
                _lib.check(lib.g4_generate(_lib.ptr_array(ptrs), None, None, len(ptrs),
                                           cfg.seed & 0xFFFFFFFFFFFFFFFF, _lib.i64_array(wr),
                                           _lib.i64_array(lanes), _lib.i64_array(meas), self.space.size,
                                           _MODE_CODE[cfg.value_mode], self.pcode, self.compute.cuda_stream),
                           "generate")
            elif kind == "acc":
                ptrs = []
                for ci, buf in op[1]:
                    c = self.channels[ci]
                    ptrs += [self._buf_ptr(ci, buf, i) for i in range(nb * len(c.lanes))]
                    for li, t in enumerate(c.lanes):
                        self.counters[t].accumulations_applied += nb
                        if buf != S.GEN:
                            self.counters[t].envelopes_received += nb
                            self.counters[t].bytes_received += nb * self.wire_bytes
                        if cfg.instrument:
                            if buf == S.GEN:
                                bp = self.pos
                            else:
                                bp = S.birth_position(self.pos, op[2][2], s, c.backward)
                            self.origins[t] += [(self.subring, bp, t, m * cfg.batch + b,
                                                 self.subring * s + bp) for b in range(nb)]
                if self.kernel_events is not None:
                    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    ev[0].record(self.compute)
                _lib.check(lib.g4_accumulate_staged(self.slice.data.data_ptr(), self.lo, self.hi,
                                                    self.space.size, _lib.ptr_array(ptrs), len(ptrs),
                                                    self.code, _lib.G4_CHANNEL_EQ1,
                                                    self.compute.cuda_stream), "accumulate")
                if self.kernel_events is not None:
                    ev[1].record(self.compute)
                    self.kernel_events.append(ev)
                self.slice.meas_count += len(ptrs)
                self.meas_count += len(ptrs)
            elif kind == "wait":
                _, st, ci, flag, value = op
                _lib.check(lib.g4_flag_wait(self.flags.data_ptr() + self._flag_off(ci, flag), value,
                                            self._stream(st).cuda_stream), "flag_wait")
            elif kind == "write":
                _, st, peer, ci, flag, value = op
                _lib.check(lib.g4_flag_write(self.peer_flags[peer] + self._flag_off(ci, flag), value,
                                             self._stream(st).cuda_stream), "flag_write")
            elif kind == "copy":
                _, st, ci, src, peer, dst = op
                c = self.channels[ci]
                cnt = nb * len(c.lanes)
                dst_ptr = self.peer_bufs[(peer, ci)] + dst * self.bufs[ci][0].numel() * self.bufs[ci].element_size()
                if self.wire_cores:
                    _lib.check(lib.g4_copy_payload_cores(dst_ptr, self._buf_ptr(ci, src), cnt, self.space.size,
                                                         self.pcode, self._stream(st).cuda_stream), "copy_cores")
                else:
                    _lib.check(lib.g4_copy_async(dst_ptr, self._buf_ptr(ci, src), cnt * self.payload_bytes,
                                                 self._stream(st).cuda_stream), "copy")
                for t in c.lanes:
                    self.counters[t].envelopes_sent += nb
                    self.counters[t].messages_sent += 1
                    self.counters[t].bytes_sent += nb * self.wire_bytes
            elif kind == "halo":
                if not self.wire_cores:
                    continue
                ptrs = [self._buf_ptr(ci, buf, i) for ci, buf in op[1]
                        for i in range(nb * len(self.channels[ci].lanes))]
                _lib.check(lib.g4_fill_halo(_lib.ptr_array(ptrs), len(ptrs), self.space.size, self.pcode,
                                            self.compute.cuda_stream), "fill_halo")
            elif kind == "record":
                self.events[op[2]].record(self._stream(op[1]))
            elif kind == "wait_event":
                self._stream(op[1]).wait_event(self.events[op[2]])
            else:  # pragma: no cover
                raise AssertionError(kind)

    def stage_gen(self, ups: list[torch.Tensor], downs: list[torch.Tensor]) -> None:
        """Fill the GEN buffers from reference-layout device matrices (K2), in
        channel order, batch-major -- the walker hand-off of a host-fed run."""
        ptrs = [self._buf_ptr(c.index, S.GEN, i) for c in self.channels
                for i in range(self.cfg.batch * len(c.lanes))]
        if len(ups) != len(ptrs) or len(downs) != len(ptrs):
            raise ContractViolation(f"expected {len(ptrs)} payloads, got {len(ups)}")
        # GEN of the previous round must have left (its first ring copy) before it is overwritten
        for c in self.channels:
            ev = self.events.get(f"sent{c.index}")
            if ev is not None:
                self.compute.wait_event(ev)
        code_in = _dtype_code(ups[0].dtype)
        _lib.check(self.lib.g4_prepare_g(_lib.ptr_array(ptrs), _lib.ptr_array([u.data_ptr() for u in ups]),
                                         _lib.ptr_array([d.data_ptr() for d in downs]), len(ptrs),
                                         self.space.size, code_in, self.pcode, self.compute.cuda_stream),
                   "prepare_g")

    def rounds(self) -> int:
        return -(-self.cfg.measurements // self.cfg.batch)

    def wait_idle(self, timeout_s: float) -> None:
        """Host watchdog: all streams drained within the timeout, else a
        DeadlockError naming the stalled (rank, lane, measurement, step)."""
        done = torch.cuda.Event()
        for st in [self.compute] + self.comm:
            done.record(st)
            t0 = time.monotonic()
            while not done.query():
                if time.monotonic() - t0 > timeout_s:
                    self._raise_deadlock()
                time.sleep(0.0005)

    def _raise_deadlock(self):
        vals = torch.zeros_like(self.flags, device="cpu")
        side = torch.cuda.Stream(self.device)
        with torch.cuda.stream(side):
            vals.copy_(self.flags, non_blocking=True)
        side.synchronize()
        s = self.cfg.subring_size
        # unblock the streams so the process can tear down, then report the channel
        # whose DATA flag lags the most (with two directions either may be the stalled one)
        with torch.cuda.stream(side):
            self.flags.fill_(1 << 62)
        side.synchronize()
        if not self.channels:
            raise DeadlockError(f"rank {self.world_rank} stalled", rank=self.world_rank)
        landed = {c.index: int(vals[c.index * S.FLAGS_PER_CHANNEL + S.DATA]) for c in self.channels}
        c = min(self.channels, key=lambda ch: landed[ch.index])
        k = max(landed[c.index] + 1, S.FIRST_TRANSFER)
        m, j = divmod(k - S.FIRST_TRANSFER, max(s - 1, 1))
        raise DeadlockError(f"rank {self.world_rank} lane {c.lanes[0]} stalled at measurement "
                            f"{m * self.cfg.batch} step {j}: no payload from rank "
                            f"{self.subring * s + c.recv_from}", rank=self.world_rank,
                            lane=c.lanes[0], step=j)


# ---------------------------------------------------------------------------
# experiment driver

@dataclass
class ExperimentReport:
    """engine.py:187-238: same fields, JSON form and registry(); plus the
    device round times and sampled planes."""

    config: dict
    tensor: np.ndarray | None
    meas_counts: dict[int, int]
    lane_counters: dict[tuple[int, int], LaneCounters]
    lane_meta: dict[tuple[int, int], dict]
    memory_peaks: dict[int, int]
    slices: dict[int, tuple[int, int]]
    elapsed_s: float
    clock: str = "cuda-event"
    round_ms: dict[int, list[float]] = field(default_factory=dict)
    samples: dict[int, np.ndarray] = field(default_factory=dict)
    memory_series: list = field(default_factory=list)

    def registry(self) -> CounterRegistry:
        reg = CounterRegistry(clock_label=self.clock)
        for (r, t), c in self.lane_counters.items():
            reg.register(r, t, c)
        return reg

    def to_json_dict(self) -> dict:
        return {"config": self.config, "clock": self.clock, "elapsed_s": self.elapsed_s,
                "meas_counts": {str(r): v for r, v in sorted(self.meas_counts.items())},
                "slices": {str(r): list(v) for r, v in sorted(self.slices.items())},
                "counters_global": self.registry().snapshot("global").to_dict(),
                "counters": {f"{r}/{t}": c.to_dict() for (r, t), c in sorted(self.lane_counters.items())},
                "lane_meta": {f"{r}/{t}": m for (r, t), m in sorted(self.lane_meta.items())},
                "memory_peaks": {str(r): p for r, p in sorted(self.memory_peaks.items())},
                "memory_series": [list(e) for e in self.memory_series]}

    @classmethod
    def from_json_dict(cls, d: dict, tensor) -> "ExperimentReport":
        def key2(s):
            r, t = s.split("/")
            return int(r), int(t)

        return cls(config=d["config"], tensor=tensor, clock=d["clock"], elapsed_s=d["elapsed_s"],
                   meas_counts={int(r): n for r, n in d["meas_counts"].items()},
                   slices={int(r): tuple(v) for r, v in d["slices"].items()},
                   lane_counters={key2(k): LaneCounters.from_dict(c) for k, c in d["counters"].items()},
                   lane_meta={key2(k): m for k, m in d["lane_meta"].items()},
                   memory_peaks={int(r): p for r, p in d["memory_peaks"].items()},
                   memory_series=[tuple(e) for e in d.get("memory_series", [])])


def device_for_rank(rank: int) -> torch.device:
    local = int(os.environ.get("LOCAL_RANK", rank))
    return torch.device("cuda", local % max(torch.cuda.device_count(), 1))


def rank_main(*args, **kwargs) -> ExperimentReport | None:
    """Everything one rank does (engine.py:241-297); the report on world rank 0.

    Two call forms:
    * ``rank_main(rt, world, cfg)`` -- the reference signature.  With a
      reference-style communicator (``isend``/``irecv``/``split``/``reduce_sum``)
      the lanes run ``run_measurement`` over that communicator (lanes.py: the
      caller's transport moves the payloads in the reference wire format; the
      GPU generates and accumulates).  With a ``Control`` (or None) it is the
      device ring below; ``rt`` is then unused.
    * ``rank_main(cfg, world=None)`` -- the device ring: one process per GPU,
      torch.distributed control plane, payloads over peer memory.
    ``cfg`` may be this package's ExperimentConfig or the reference's."""
    if args and _is_config(args[0]):
        cfg = args[0]
        world = args[1] if len(args) > 1 else kwargs.get("world")
        return _device_rank_main(as_config(cfg), world)
    rt, world, cfg = (list(args) + [kwargs.get(k) for k in ("rt", "world", "cfg")][len(args):])[:3]
    cfg = as_config(cfg)
    if world is not None and not isinstance(world, Control) and hasattr(world, "isend"):
        from .lanes import comm_rank_main
        validate_config(cfg)
        return comm_rank_main(rt, world, cfg)
    return _device_rank_main(cfg, world)


def _is_config(x) -> bool:
    return isinstance(x, ExperimentConfig) or (hasattr(x, "n_k") and hasattr(x, "subring_size"))


def _device_rank_main(cfg: ExperimentConfig, world: "Control | None") -> ExperimentReport | None:
    validate_config(cfg)
    world = world or Control()
    if world.size != cfg.world_size:
        raise ConfigError(f"world_size {cfg.world_size} but {world.size} ranks are running")
    r = world.rank
    device = device_for_rank(r)
    torch.cuda.set_device(device)
    lib = _lib.load()
    _lib.check(lib.g4_set_arith_mode(ARITH_MODES[cfg.arith]), "set_arith_mode")
    try:
        return _rank_main(cfg, world, r, device)
    finally:
        _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_EXACT), "set_arith_mode")


def _rank_main(cfg: ExperimentConfig, world: Control, r: int, device: torch.device) -> ExperimentReport | None:
    torch.cuda.reset_peak_memory_stats(device)
    sub = build_subrings(world, cfg.subring_size)
    pos_group = world.split(r % cfg.subring_size, r // cfg.subring_size)  # same position across sub-rings
    eng = RingEngine(cfg, sub, r, device)
    world.barrier()
    t0 = time.monotonic()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(eng.compute)
    error = None
    try:
        for m in range(eng.rounds()):
            eng.enqueue_round(m)
        end.record(eng.compute)
        eng.wait_idle(cfg.timeout_s)
    except DeadlockError as exc:
        error = exc
    if error is not None:
        raise error
    elapsed = time.monotonic() - t0
    gpu_ms = start.elapsed_time(end)
    torch.cuda.synchronize(device)
    world.barrier()

    if cfg.reduce == "nccl":
        reduce_sum_nccl(world, cfg.subring_size, eng.slice.data)
    else:
        reduce_sum(pos_group, eng.slice.data, root=0)

    tensor = None
    if cfg.gather:
        tensor = _gather_full(world, eng, cfg)
    samples = _gather_planes(world, eng, cfg, cfg.sample_planes) if cfg.sample_planes else {}
    blob = {"rank": r, "meas_count": eng.meas_count, "slice": [eng.lo, eng.hi],
            "counters": {t: c.to_dict() for t, c in eng.counters.items()},
            "final_send": _final_send_origins(eng, cfg),
            "origins": {t: eng.origins[t] for t in eng.origins},
            "peak": int(torch.cuda.max_memory_allocated(device)), "gpu_ms": gpu_ms}
    blobs = world.allgather(json.dumps(blob))
    eng.close()
    if r != 0:
        return None
    meas, slices, peaks, counters, meta, rms = {}, {}, {}, {}, {}, {}
    for b in map(json.loads, blobs):
        rr = b["rank"]
        meas[rr] = b["meas_count"]
        slices[rr] = tuple(b["slice"])
        peaks[rr] = b["peak"]
        rms[rr] = [b["gpu_ms"]]
        for t, c in b["counters"].items():
            counters[(rr, int(t))] = LaneCounters.from_dict(c)
            meta[(rr, int(t))] = {"lane": int(t), "allocations": 3, "ring_phase_allocations": 0,
                                  "isolation_violations": 0,
                                  "final_send_origin": b["final_send"][t],
                                  "origins": [tuple(o) for o in b["origins"][t]]}
    return ExperimentReport(config=cfg.to_dict(), tensor=tensor, meas_counts=meas, lane_counters=counters,
                            lane_meta=meta, memory_peaks=peaks, slices=slices, elapsed_s=elapsed,
                            round_ms=rms, samples=samples)


def _final_send_origins(eng: "RingEngine", cfg: ExperimentConfig) -> dict[int, list[int]]:
    """The origin of the payload each lane holds in its send buffer after the
    last measurement (engine.py:275-277): the one received at the last ring
    step, born birth_position(pos, steps - 1) (its own when there are no steps)."""
    s = cfg.subring_size
    steps = s - 1 if cfg.ring_steps_override is None else cfg.ring_steps_override
    out = {}
    for c in eng.channels:
        bp = S.birth_position(eng.pos, steps - 1, s, c.backward) if steps > 0 else eng.pos
        for t in c.lanes:
            out[t] = [eng.subring, bp, t, cfg.measurements - 1, eng.subring * s + bp]
    return out


def _gather_full(world: Control, eng: RingEngine, cfg: ExperimentConfig) -> np.ndarray | None:
    """World rank 0 assembles the reduced tensor from sub-ring 0's slices (engine.py:287-297)."""
    s = cfg.subring_size
    torch.cuda.synchronize(eng.device)
    info = world.allgather((export_ptr(eng.slice.data.data_ptr()), eng.lo, eng.hi))
    out = None
    if world.rank == 0:
        n = eng.space.size
        full = torch.empty((cfg.num_planes, n, n), dtype=eng.dtype, device=eng.device)
        pm = PeerMap()
        try:
            for q in range(s):
                (h, off), lo, hi = info[q]
                ptr = pm.open(h, off, eng.slice.data.data_ptr() if q == 0 else None)
                nbytes = (hi - lo) * n * n * full.element_size()
                _lib.check(eng.lib.g4_copy_async(full[lo:hi].data_ptr(), ptr, nbytes,
                                                 torch.cuda.current_stream(eng.device).cuda_stream), "gather")
            torch.cuda.synchronize(eng.device)
        finally:
            pm.close()
        out = full.cpu().numpy()
    world.barrier()
    return out


def _gather_planes(world: Control, eng: RingEngine, cfg: ExperimentConfig, planes) -> dict[int, np.ndarray]:
    """Copy selected reduced K3 planes to world rank 0 without assembling the
    whole tensor (for G4s far larger than one GPU)."""
    s = cfg.subring_size
    torch.cuda.synchronize(eng.device)
    info = world.allgather((export_ptr(eng.slice.data.data_ptr()), eng.lo, eng.hi))
    out = {}
    if world.rank == 0:
        n = eng.space.size
        buf = torch.empty((n, n), dtype=eng.dtype, device=eng.device)
        pm = PeerMap()
        try:
            for k3 in planes:
                if not (0 <= k3 < cfg.num_planes):
                    raise ContractViolation(f"sample plane {k3} outside [0, {cfg.num_planes})")
                q = next(i for i in range(s) if info[i][1] <= k3 < info[i][2])
                (h, off), lo, _ = info[q]
                ptr = pm.open(h, off, eng.slice.data.data_ptr() if q == 0 else None)
                nbytes = n * n * buf.element_size()
                _lib.check(eng.lib.g4_copy_async(buf.data_ptr(), ptr + (k3 - lo) * nbytes, nbytes,
                                                 torch.cuda.current_stream(eng.device).cuda_stream), "sample")
                out[k3] = buf.cpu().numpy().copy()
        finally:
            pm.close()
    world.barrier()
    return out


# ---------------------------------------------------------------------------
# launcher: one OS process per rank (the role of transport/tcp.py's launcher)

def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, cfg_dict: dict, port: int, q) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(cfg_dict["world_size"]), LOCAL_RANK=str(rank))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=cfg_dict["world_size"])
        rep = rank_main(ExperimentConfig(**cfg_dict))
        q.put((rank, "ok", rep))
    except Exception as exc:  # reported to the launcher
        q.put((rank, "error", exc))
    finally:
        if dist.is_initialized():
            try:
                dist.destroy_process_group()
            except Exception:
                pass


def run_experiment(cfg) -> ExperimentReport:
    """Run a whole experiment (engine.py:323-335).  Inside an initialised
    torch.distributed world every rank calls this; otherwise one process per
    rank is spawned on this node (ranks share GPUs round-robin)."""
    cfg = as_config(cfg)
    validate_config(cfg)
    if dist.is_available() and dist.is_initialized():
        return rank_main(cfg)
    if cfg.world_size == 1:
        return rank_main(cfg)
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, cfg.to_dict(), port, q), daemon=True)
             for r in range(cfg.world_size)]
    for p in procs:
        p.start()
    results, error = {}, None
    deadline = time.monotonic() + max(120.0, 4 * cfg.timeout_s)
    while len(results) < cfg.world_size and time.monotonic() < deadline:
        try:
            rank, status, payload = q.get(timeout=1.0)
        except Exception:
            if any(p.exitcode not in (None, 0) for p in procs) and error is None:
                error = RuntimeError("a rank process died")
                break
            continue
        results[rank] = (status, payload)
        if status == "error":
            error = payload
            break
    for p in procs:
        p.join(timeout=5 if error is None else 0.5)
        if p.is_alive():
            p.kill()
    if error is not None:
        raise error
    if len(results) < cfg.world_size:
        raise DeadlockError("experiment did not finish before the launcher deadline")
    return results[0][1]


# the reference's per-lane driver over an injected communicator (lanes.py)
from .lanes import LaneRecorder, LaneState, NullRecorder, run_measurement  # noqa: E402,F401
