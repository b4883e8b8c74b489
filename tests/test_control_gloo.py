"""Control plane of the ring driver on CPU: communicator split / sub-ring
construction over torch.distributed gloo with several processes
(reference tests/test_engine.py:56-81, TestBuildSubrings)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2105_00027_b200.errors import ConfigError


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn_name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_00027_b200 import engine as E
        ctl = E.Control()
        q.put((rank, globals()[fn_name](E, ctl)))
    except Exception as exc:
        q.put((rank, exc))
    finally:
        dist.destroy_process_group()


def run_ranks(world, fn_name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn_name, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(30)
    return out


def subring_of_3(E, ctl):
    s = E.build_subrings(ctl, 3)
    return (s.size, s.rank, s.world_ranks)


def subring_of_4_positions(E, ctl):
    s = E.build_subrings(ctl, 4)
    pos = ctl.split(ctl.rank % 4, ctl.rank // 4)
    return (s.rank, s.world_ranks, pos.rank, pos.world_ranks, s.allgather(ctl.rank))


def indivisible(E, ctl):
    try:
        E.build_subrings(ctl, 4)
    except ConfigError:
        return "ConfigError"
    return "no error"


def test_consecutive_grouping():
    out = run_ranks(6, "subring_of_3")
    assert out[0] == (3, 0, (0, 1, 2)) and out[5] == (3, 2, (3, 4, 5))


def test_subrings_and_position_groups():
    out = run_ranks(8, "subring_of_4_positions")
    for r, (srank, members, prank, pmembers, gathered) in out.items():
        assert srank == r % 4 and members == tuple(range(r - r % 4, r - r % 4 + 4))
        assert prank == r // 4 and pmembers == (r % 4, r % 4 + 4)
        assert gathered == list(members)  # allgather inside the sub-ring, rank order


def test_indivisible_rejected():
    out = run_ranks(6, "indivisible")
    assert set(out.values()) == {"ConfigError"}
