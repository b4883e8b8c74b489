"""The native ring driver of the C ABI (g4_ring_create / measure / wait /
reduce / destroy): the host a cgo/JNI/C++ caller would use, driven here from
Python through ctypes with a gloo all-gather as its control plane.  Several
rank processes share the test box's GPU(s).  Results are compared with the
oracle's serial sum over every walker of every lane and sub-ring (the
reference run_experiment's tensor).  GPU only.
"""
import ctypes
import os
import queue
import time

import numpy as np
import pytest

from oracle import oracle as O
from paper_2105_00027_b200 import _lib

pytestmark = pytest.mark.gpu


def _worker(rank, world, cfgd, port, q, skip_rank):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(rank % torch.cuda.device_count())
        S = cfgd["subring_size"]
        sub = [dist.new_group([g * S + i for i in range(S)]) for g in range(world // S)]
        pos = [dist.new_group([p + g * S for g in range(world // S)]) for p in range(S)]
        groups = {_lib.G4_GROUP_SUBRING: sub[rank // S], _lib.G4_GROUP_POSITION: pos[rank % S]}

        def allgather(ctx, group, send, nbytes, recv):
            try:
                grp = groups[group]
                out = [None] * dist.get_world_size(grp)
                dist.all_gather_object(out, ctypes.string_at(send, nbytes), group=grp)
                ctypes.memmove(recv, b"".join(out), nbytes * len(out))
                return 0
            except Exception:  # pragma: no cover - reported as G4_ERR_TRANSPORT
                return 1

        cb = _lib.ALLGATHER_FN(allgather)
        lib = _lib.load()
        cfg = _lib.RingConfig(**{k: v for k, v in cfgd.items() if k != "rounds"})
        ring = ctypes.c_void_p()
        _lib.check(lib.g4_ring_create(ctypes.byref(cfg), rank, cb, None, ctypes.byref(ring)), "ring_create")
        err = None
        if rank != skip_rank:
            for m in range(cfgd["rounds"]):
                _lib.check(lib.g4_ring_measure(ring, m, 1), "ring_measure")
            try:
                _lib.check(lib.g4_ring_wait(ring, 5000 if skip_rank >= 0 else 120000), "ring_wait")
            except Exception as exc:  # DeadlockError in the negative control
                err = exc
        if err is None and skip_rank < 0:
            _lib.check(lib.g4_ring_reduce(ring), "ring_reduce")
        data, lo, hi = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(lib.g4_ring_slice(ring, ctypes.byref(data), ctypes.byref(lo), ctypes.byref(hi)), "ring_slice")
        n = cfgd["n_k"] * cfgd["n_w"]
        dt = torch.complex64 if cfgd["dtype"] == _lib.G4_C64 else torch.complex128
        dev = torch.empty((hi.value - lo.value, n, n), dtype=dt, device="cuda")
        torch.cuda.synchronize()
        _lib.check(lib.g4_copy_async(dev.data_ptr(), data, dev.numel() * dev.element_size(), None), "copy")
        torch.cuda.synchronize()
        _lib.check(lib.g4_ring_destroy(ring), "ring_destroy")
        q.put((rank, "ok", (lo.value, hi.value, dev.cpu().numpy(),
                            None if err is None else (type(err).__name__, str(err)))))
    except Exception as exc:  # pragma: no cover
        q.put((rank, "error", repr(exc)))


def run_native(cfgd, skip_rank=-1):
    import torch.multiprocessing as tmp
    from paper_2105_00027_b200.engine import _free_port
    world = cfgd["world_size"]
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, cfgd, port, q, skip_rank), daemon=True)
             for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    deadline = time.monotonic() + 300
    while len(out) < world and time.monotonic() < deadline:
        try:
            r, status, payload = q.get(timeout=1.0)
        except queue.Empty:
            continue
        assert status == "ok", payload
        out[r] = payload
    for p in procs:
        p.join(timeout=10)
    assert len(out) == world, "rank processes did not finish"
    return out


def config(**kw):
    d = dict(n_k=2, n_w=4, world_size=2, subring_size=2, lanes=1, alternate=0, batch=2, dtype=_lib.G4_C128,
             planes=0, value_mode=_lib.G4_MODE_INTEGER, reserved=0, seed=11, rounds=2)
    d.update(kw)
    return d


@pytest.mark.parametrize("kw", [
    dict(),
    dict(world_size=1, subring_size=1, lanes=2, rounds=3),
    dict(world_size=4, subring_size=2, lanes=2, alternate=1, batch=1, rounds=3),      # 2 sub-rings + reduce
    dict(world_size=3, subring_size=3, lanes=3, alternate=1, n_w=3, batch=1, rounds=2),
    dict(world_size=4, subring_size=4, lanes=1, n_k=8, n_w=16, planes=64, batch=4, rounds=3,
         value_mode=_lib.G4_MODE_FLOAT),                                               # K1 v2 path
])
def test_native_ring_matches_oracle(kw):
    c = config(**kw)
    res = run_native(c)
    n = c["n_k"] * c["n_w"]
    planes = c["planes"] or n
    S = c["subring_size"]
    full = np.zeros((planes, n, n), np.complex128)
    for r in range(S):  # sub-ring 0 holds the reduced tensor
        lo, hi, data, err = res[r]
        assert err is None
        full[lo:hi] = data
    mode = "integer" if c["value_mode"] == _lib.G4_MODE_INTEGER else "float"
    ref = O.oracle_full(c["seed"], n, c["world_size"] // S, S, c["lanes"], c["rounds"] * c["batch"], mode, 0,
                        planes)
    if mode == "integer":
        assert np.array_equal(full, ref)
    else:
        np.testing.assert_allclose(full, ref, rtol=1e-10, atol=1e-10 * np.abs(ref).max())


def test_native_ring_deadlock_diagnostic():
    """Negative control: rank 1 never runs its rounds, so rank 0 starves."""
    res = run_native(config(rounds=1), skip_rank=1)
    err = res[0][3]
    assert err is not None and err[0] == "DeadlockError"
    assert "rank 0" in err[1] and "lane 0" in err[1] and "no payload from rank 1" in err[1]
