"""A reference-style in-process communicator and runtime for tests (test
infrastructure, no product code): the surface of ringacc.transport.base
(Communicator: rank/size/world_ranks, isend/irecv with tagged FIFO matching,
split by (color, key, parent rank), reduce_sum in canonical rank order) and of
an in-process Runtime (spawn/join/now/make_lock), written from that contract
so the communicator path of ``engine.rank_main(rt, world, cfg)`` can be
tested on the GPU box, where the reference package is absent.
"""
from __future__ import annotations

import pickle
import queue
import threading
import time

import numpy as np

from paper_2105_00027_b200.errors import ContractViolation, DeadlockError


class Hub:
    def __init__(self, world_size: int, timeout_s: float = 10.0):
        self.world_size = world_size
        self.timeout_s = timeout_s
        self._q: dict[tuple, queue.Queue] = {}
        self._lock = threading.Lock()
        self._ctx = 0

    def chan(self, key) -> queue.Queue:
        with self._lock:
            return self._q.setdefault(key, queue.Queue())

    def new_ctx(self) -> int:
        with self._lock:
            self._ctx += 1
            return self._ctx

    def comm(self, rank: int) -> "Comm":
        return Comm(self, 0, rank, tuple(range(self.world_size)))


class _Done:
    def wait(self, timeout=None):
        return None


class _Recv:
    def __init__(self, q, timeout, src, tag):
        self.q, self.timeout, self.src, self.tag = q, timeout, src, tag

    def wait(self, timeout=None):
        try:
            return self.q.get(timeout=timeout or self.timeout)
        except queue.Empty:
            raise DeadlockError(f"receive from rank {self.src} tag {self.tag} timed out") from None


class Comm:
    SYS = 1 << 40

    def __init__(self, hub: Hub, ctx: int, rank: int, world_ranks: tuple[int, ...]):
        self.hub, self.ctx, self.rank, self.world_ranks = hub, ctx, rank, world_ranks
        self.size = len(world_ranks)
        self._seq = 0

    def isend(self, dest, tag, payload):
        if not 0 <= dest < self.size:
            raise ContractViolation(f"send dest rank {dest} outside [0, {self.size})")
        self.hub.chan((self.ctx, self.rank, dest, tag)).put(bytes(payload))
        return _Done()

    def irecv(self, src, tag):
        if not 0 <= src < self.size:
            raise ContractViolation(f"recv source rank {src} outside [0, {self.size})")
        return _Recv(self.hub.chan((self.ctx, src, self.rank, tag)), self.hub.timeout_s, src, tag)

    def _tag(self) -> int:
        self._seq += 1
        return self.SYS + self._seq

    def split(self, color: int, key: int) -> "Comm":
        tag = self._tag()
        if self.rank == 0:
            entries = [(color, key, 0)] + [pickle.loads(self.irecv(r, tag).wait()) + (r,)
                                           for r in range(1, self.size)]
            groups: dict[int, list] = {}
            for c, k, r in entries:
                groups.setdefault(c, []).append((k, r))
            replies = {}
            for c, members in groups.items():
                ctx = self.hub.new_ctx()
                parents = [r for _, r in sorted(members)]
                for i, pr in enumerate(parents):
                    replies[pr] = (ctx, i, parents)
            for r in range(1, self.size):
                self.isend(r, tag, pickle.dumps(replies[r]))
            ctx, me, parents = replies[0]
        else:
            self.isend(0, tag, pickle.dumps((color, key)))
            ctx, me, parents = pickle.loads(self.irecv(0, tag).wait())
        return Comm(self.hub, ctx, me, tuple(self.world_ranks[p] for p in parents))

    def reduce_sum(self, local, root: int = 0):
        tag = self._tag()
        mine = np.asarray(local, dtype=np.complex128)
        if self.rank != root:
            self.isend(root, tag, pickle.dumps(mine))
            return None
        total = None
        for r in range(self.size):
            arr = mine if r == self.rank else pickle.loads(self.irecv(r, tag).wait())
            total = arr.copy() if total is None else total + arr
        return total


class _Handle:
    def __init__(self):
        self.thread = None
        self.error = None


class Runtime:
    clock_label = "monotonic"

    def __init__(self):
        self._t0 = time.perf_counter()

    def now(self) -> float:
        return time.perf_counter() - self._t0

    def make_lock(self):
        return threading.Lock()

    def spawn(self, fn, *args, name=None):
        h = _Handle()

        def run():
            try:
                fn(*args)
            except BaseException as exc:
                h.error = exc
        h.thread = threading.Thread(target=run, name=str(name), daemon=True)
        h.thread.start()
        return h

    def join(self, handles):
        for h in handles:
            h.thread.join()
        errs = [h.error for h in handles if h.error is not None]
        for e in errs:
            if isinstance(e, DeadlockError) and e.step is not None:
                raise e
        if errs:
            raise errs[0]


def run_world(cfg, rank_main, timeout_s: float = 10.0):
    """Every rank of `cfg` as a thread calling rank_main(rt, world, cfg); the
    rank-0 report."""
    hub = Hub(cfg.world_size, timeout_s)
    rt = Runtime()
    out = {}

    def entry(r):
        out[r] = rank_main(rt, hub.comm(r), cfg)
    rt.join([rt.spawn(entry, r, name=(r, None)) for r in range(cfg.world_size)])
    return out[0]
