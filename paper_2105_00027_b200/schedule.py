"""Ring topology and the per-rank operation schedule of one measurement round.

Host logic only (no CUDA): mirrors the reference ring semantics of
``ringacc/engine.py`` and turns them into an explicit list of stream-ordered
operations that ``engine.py`` executes on a B200 (copy engine + stream flags +
K1/K3 kernels) and that the CPU tests execute with a host simulator.

Reference semantics kept (engine.py:40-161):
  * sub-ring neighbours left = (r - 1) mod S, right = (r + 1) mod S;
  * lane tag = 1000 + lane, lanes < 1000; ``alternate`` reverses odd lanes;
  * per measurement every lane accumulates its own payload, then for exactly
    S - 1 steps forwards the payload it holds to the right and accumulates the
    one received from the left; each payload ends at the left neighbour of its
    birth rank; three payload buffers per lane, no allocation in the ring phase.

B200 realisation (one round = B measurements of every lane):
  * lanes sharing a direction form one *channel*; a channel's payloads for the
    round travel together (one copy per ring step), so all lanes' payloads of a
    step are applied in ONE K1 pass;
  * per channel and rank: buffers GEN (own payloads), R0, R1 (receive slots) and
    three 64-bit flags living on that rank: DATA (written by the left neighbour:
    index of the last transfer that landed here), ACK_ACC and ACK_FWD (written
    by the right neighbour: last transfer it has accumulated / forwarded).
  * transfer k (k = 2 + m*(S-1) + j for round m, step j) lands in slot k % 2 of
    the receiver; before sending it the sender waits until the receiver has
    both accumulated and forwarded transfer k - 2 (which occupied that slot).
  * only the N x N payload cores cross the link; the receiver rebuilds the
    staged layout's halo on its compute stream before K1 reads the slot.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

from .errors import ConfigError, ContractViolation

RECV_TAG = 1000
SEND_TAG = 1000
MAX_LANES = 1000
FIRST_TRANSFER = 2

# buffer ids within a channel
GEN, R0, R1 = 0, 1, 2
# flag ids within a channel
DATA, ACK_ACC, ACK_FWD = 0, 1, 2
FLAGS_PER_CHANNEL = 4  # padded to 32 B

COMPUTE = "compute"


@dataclass(frozen=True)
class RingTopology:
    """Sub-ring geometry (ringacc/engine.py:40-63)."""

    world_size: int
    subring_size: int
    lanes: int
    direction: str = "forward"

    def __post_init__(self):
        if self.subring_size < 1:
            raise ConfigError("subring size must be >= 1")
        if self.world_size % self.subring_size != 0:
            raise ConfigError(f"subring size {self.subring_size} does not divide world size "
                              f"{self.world_size}")
        if not (1 <= self.lanes < MAX_LANES):
            raise ConfigError(f"lane count must be in [1, {MAX_LANES}), got {self.lanes}")
        if self.direction not in ("forward", "alternate"):
            raise ConfigError(f"unknown direction policy {self.direction!r}")

    def left(self, subring_rank: int) -> int:
        return (subring_rank - 1 + self.subring_size) % self.subring_size

    def right(self, subring_rank: int) -> int:
        return (subring_rank + 1) % self.subring_size

    @property
    def subrings(self) -> int:
        return self.world_size // self.subring_size


class LaneRing(NamedTuple):
    recv_from: int
    send_to: int
    tag: int


def lane_ring_id(topo: RingTopology, subring_rank: int, lane: int) -> LaneRing:
    """Neighbours and tag of one lane's ring (ringacc/engine.py:72-83)."""
    if lane >= topo.lanes:
        raise ContractViolation(f"lane {lane} outside [0, {topo.lanes})")
    left, right = topo.left(subring_rank), topo.right(subring_rank)
    if topo.direction == "alternate" and lane % 2 == 1:
        left, right = right, left
    return LaneRing(recv_from=left, send_to=right, tag=RECV_TAG + lane)


@dataclass(frozen=True)
class Channel:
    """Lanes of one rank that share a ring direction."""

    index: int
    lanes: tuple[int, ...]
    recv_from: int
    send_to: int
    backward: bool


def make_channels(topo: RingTopology, pos: int, per_lane: bool = False) -> list[Channel]:
    """The rank's channels: by default lanes that share a direction (same
    neighbours) share one channel -- one copy per step carries all their
    payloads.  per_lane=True gives every lane its own channel (own comm stream,
    flags and buffers), i.e. the reference's independent per-lane rings
    (engine.py:62-83) as independent device pipelines."""
    groups: dict[tuple[int, ...], list[int]] = {}
    for t in range(topo.lanes):
        ring = lane_ring_id(topo, pos, t)
        key = (ring.recv_from, ring.send_to) + ((t,) if per_lane else ())
        groups.setdefault(key, []).append(t)
    out = []
    for i, ((rf, st, *_), lanes) in enumerate(sorted(groups.items(), key=lambda kv: kv[1][0])):
        backward = topo.direction == "alternate" and lanes[0] % 2 == 1
        out.append(Channel(i, tuple(lanes), rf, st, backward))
    return out


def transfer_index(m: int, j: int, s: int) -> int:
    return FIRST_TRANSFER + m * (s - 1) + j


def birth_position(pos: int, j: int, s: int, backward: bool) -> int:
    """Sub-ring position whose payload arrives at `pos` at ring step j."""
    return (pos + 1 + j) % s if backward else (pos - 1 - j) % s


# ---- operations -------------------------------------------------------------
# Each op is a tuple whose first element is the kind:
#   ("gen", m)                                  compute: K3 fills GEN of every channel
#   ("acc", ((channel, buf), ...), tag)          compute: one K1 pass over those buffers
#   ("wait", stream, channel, flag, value)       stream blocks until my flag >= value
#   ("write", stream, peer_pos, channel, flag, value)  stream writes the flag on a neighbour
#   ("copy", stream, channel, src_buf, peer_pos, dst_buf)  copy-engine transfer of the payload cores
#   ("halo", ((channel, buf), ...))              compute: rebuild the halo of received payloads
#   ("record", stream, event) / ("wait_event", stream, event)


def comm_stream(c: Channel) -> str:
    return f"comm{c.index}"


def round_schedule(topo: RingTopology, pos: int, channels: list[Channel], m: int,
                   steps: int | None = None, skip_send_step0: bool = False) -> list[tuple]:
    """All operations of round m on sub-ring position `pos`, in enqueue order."""
    s = topo.subring_size
    steps = s - 1 if steps is None else steps
    ops: list[tuple] = []
    if m > 0 and steps > 0:
        for c in channels:  # GEN of round m-1 must have left before it is regenerated
            ops.append(("wait_event", COMPUTE, f"sent{c.index}"))
    ops.append(("gen", m))
    if steps > 0:
        ops.append(("record", COMPUTE, "gen"))
    ops.append(("acc", tuple((c.index, GEN) for c in channels), ("own", m)))
    for j in range(steps):
        k = transfer_index(m, j, s)
        for c in channels:
            cs = comm_stream(c)
            if k - 2 >= FIRST_TRANSFER:  # the slot held transfer k-2: accumulated and forwarded?
                ops.append(("wait", cs, c.index, ACK_ACC, k - 2))
                ops.append(("wait", cs, c.index, ACK_FWD, k - 2))
            if j == 0:
                ops.append(("wait_event", cs, "gen"))
                src = GEN
            else:
                ops.append(("wait", cs, c.index, DATA, k - 1))
                src = R0 + (k - 1) % 2
            if not (skip_send_step0 and j == 0 and c.index == 0):
                ops.append(("copy", cs, c.index, src, c.send_to, R0 + k % 2))
                ops.append(("write", cs, c.send_to, c.index, DATA, k))
            if j == 0:
                ops.append(("record", cs, f"sent{c.index}"))
            if j >= 1:
                ops.append(("write", cs, c.recv_from, c.index, ACK_FWD, k - 1))
            if j == steps - 1:
                ops.append(("write", cs, c.recv_from, c.index, ACK_FWD, k))
        for c in channels:
            ops.append(("wait", COMPUTE, c.index, DATA, k))
        ops.append(("halo", tuple((c.index, R0 + k % 2) for c in channels)))
        ops.append(("acc", tuple((c.index, R0 + k % 2) for c in channels), ("ring", m, j)))
        for c in channels:
            ops.append(("write", COMPUTE, c.recv_from, c.index, ACK_ACC, k))
    return ops


# Rounds 0 and 1 lack the slot-reuse waits of the steady state (their receive
# slots were never used before); from round 2 on, the schedule repeats with
# period 2 (a transfer's receive slot alternates with its index) and every
# flag value is affine in the round number.
STEADY_FROM_ROUND = 2


def steady_state_template(topo: RingTopology, pos: int, channels: list[Channel],
                          parity: int) -> list[tuple]:
    """The round schedule for every round m >= STEADY_FROM_ROUND with m % 2 ==
    parity, as one op list whose flag ops ("wait", "write") end in the pair
    (base, slope) such that the value of round m is base + slope * m.  The
    instrumentation tag of "acc" ops is dropped; "gen" ops keep no round index.
    Raises ContractViolation if the schedule is not periodic."""
    t0 = STEADY_FROM_ROUND + ((parity - STEADY_FROM_ROUND) % 2)
    rounds = [round_schedule(topo, pos, channels, t0 + 2 * i) for i in range(3)]
    if not len(rounds[0]) == len(rounds[1]) == len(rounds[2]):
        raise ContractViolation("ring schedule is not periodic in the round number")
    out = []
    for i, op in enumerate(rounds[0]):
        kind = op[0]
        key = {"acc": lambda o: o[:2], "gen": lambda o: o[:1],
               "wait": lambda o: o[:-1], "write": lambda o: o[:-1]}.get(kind, lambda o: o)
        if any(r[i][0] != kind or key(r[i]) != key(op) for r in rounds[1:]):
            raise ContractViolation("ring schedule is not periodic in the round number")
        if kind in ("wait", "write"):
            a, b, c = (r[i][-1] for r in rounds)
            if c - b != b - a or (b - a) % 2:
                raise ContractViolation("ring flag values are not affine in the round number")
            slope = (b - a) // 2
            out.append(op[:-1] + (a - slope * t0, slope))
        else:
            out.append(key(op))
    return out
