"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the G4 ring-accumulation hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference`` arm) may import this module.  The product package
``paper_2105_00027_b200`` never imports it: on a machine without the CUDA
library the product raises instead of falling back here.

Two restatements of the reference (``/root/reference/pkg/src/ringacc/tensor.py``):

* ``libg4oracle.so`` (``oracle/g4_oracle.c``), plain C, one entry at a time with
  the reference's exact floating-point op order.  This is the parity checker.
* ``accumulate_np`` below, a numpy port of ``accumulate_g4`` (tensor.py:233-251)
  with the same gather/multiply/transpose-add structure; it is the CPU baseline
  ("kind": "port") that bench.py times on the GPU box's host cores.

Pinning: tests/test_oracle.py checks both against golden vectors written by
oracle/make_golden.py, which imports the real reference.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libg4oracle.so"
_lib = None

FLOAT, INTEGER = 0, 1
MODES = {"float": FLOAT, "integer": INTEGER}


def build() -> Path:
    """Compile oracle/libg4oracle.so with oracle/Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        u64, i64, i32, vp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
        L.g4o_mix64.argtypes, L.g4o_mix64.restype = [u64], u64
        L.g4o_stream_key.argtypes, L.g4o_stream_key.restype = [u64, i64, i64, i64, i64], u64
        L.g4o_fill_gsigma.argtypes = [u64, i64, i64, i64, i32, i32, vp, vp]
        L.g4o_fill_gsigma.restype = None
        L.g4o_accumulate.argtypes = [vp, i64, i64, i32, vp, vp]
        L.g4o_accumulate.restype = None
        L.g4o_accumulate_c64.argtypes = [vp, i64, i64, i32, vp, vp]
        L.g4o_accumulate_c64.restype = None
        L.g4o_index_diff.argtypes, L.g4o_index_diff.restype = [i64, i64, i64], i64
        L.g4o_partition.argtypes, L.g4o_partition.restype = [i64, i64, vp], i32
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags.c_contiguous
    return ctypes.c_void_p(a.ctypes.data)


def mix64(z: int) -> int:
    return lib().g4o_mix64(z & 0xFFFFFFFFFFFFFFFF)


def stream_key(seed, world_rank, lane, meas, matrix) -> int:
    return lib().g4o_stream_key(seed, world_rank, lane, meas, matrix)


def gsigma(seed: int, world_rank: int, lane: int, meas: int, n: int,
           mode: str = "float") -> tuple[np.ndarray, np.ndarray]:
    """(up, down) for Origin(world_rank, lane, meas) -- tensor.py:215-228."""
    up = np.empty((n, n), np.complex128)
    down = np.empty((n, n), np.complex128)
    lib().g4o_fill_gsigma(seed, world_rank, lane, meas, n, MODES[mode], _ptr(up), _ptr(down))
    return up, down


def accumulate(g4: np.ndarray, lo: int, hi: int, up: np.ndarray, down: np.ndarray) -> None:
    """In-place C oracle of accumulate_g4 on planes [lo, hi).  complex128 or complex64."""
    n = up.shape[0]
    assert g4.shape == (hi - lo, n, n) and up.shape == down.shape == (n, n)
    if g4.dtype == np.complex128:
        u = np.ascontiguousarray(up, np.complex128)
        d = np.ascontiguousarray(down, np.complex128)
        lib().g4o_accumulate(_ptr(g4), lo, hi, n, _ptr(u), _ptr(d))
    elif g4.dtype == np.complex64:
        u = np.ascontiguousarray(up, np.complex64)
        d = np.ascontiguousarray(down, np.complex64)
        lib().g4o_accumulate_c64(_ptr(g4), lo, hi, n, _ptr(u), _ptr(d))
    else:
        raise TypeError(g4.dtype)


def index_diff(a: int, b: int, n: int) -> int:
    return lib().g4o_index_diff(a, b, n)


def partition(n: int, p: int) -> tuple[tuple[int, int], ...]:
    out = np.zeros(2 * max(p, 1), np.int64)
    if lib().g4o_partition(n, p, _ptr(out)) != 0:
        raise ValueError(f"cannot split {n} over {p}")
    return tuple((int(out[2 * i]), int(out[2 * i + 1])) for i in range(p))


def accumulate_np(g4: np.ndarray, lo: int, hi: int, up: np.ndarray, down: np.ndarray) -> None:
    """numpy port of accumulate_g4 (tensor.py:246-250): per plane, gather the
    cyclically shifted operands, form u*down + d*up and add its transpose."""
    n = up.shape[0]
    cols = np.arange(n)
    for k3 in range(lo, hi):
        sh = (k3 - cols) % n
        u = up.take(sh, axis=0).take(sh, axis=1)
        d = down.take(sh, axis=0).take(sh, axis=1)
        g4[k3 - lo] += (u * down + d * up).T


def brute_force(up: np.ndarray, down: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """Literal per-entry loop of Eq. 1 for tiny N (mirrors the reference's
    independent test oracle, tests/test_tensor.py:12-24)."""
    n = up.shape[0]
    out = np.zeros((hi - lo, n, n), np.complex128)
    for k3 in range(lo, hi):
        for k1 in range(n):
            for k2 in range(n):
                a, b = (k3 - k2) % n, (k3 - k1) % n
                out[k3 - lo, k1, k2] = up[a, b] * down[k2, k1] + down[a, b] * up[k2, k1]
    return out


def origins(subrings: int, subring_size: int, lanes: int, measurements: int):
    """Canonical origin order (tensor.py:265-273): (subring, rank, lane, meas, world_rank)."""
    return [(s, r, t, m, s * subring_size + r)
            for s in range(subrings) for r in range(subring_size)
            for t in range(lanes) for m in range(measurements)]


def oracle_full(seed: int, n: int, subrings: int, subring_size: int, lanes: int,
                measurements: int, mode: str = "float", lo: int = 0, hi: int | None = None,
                dtype=np.complex128) -> np.ndarray:
    """Serial ground truth (tensor.py:276-283) restricted to planes [lo, hi)."""
    hi = n if hi is None else hi
    out = np.zeros((hi - lo, n, n), dtype)
    for (_s, _r, t, m, wr) in origins(subrings, subring_size, lanes, measurements):
        up, down = gsigma(seed, wr, t, m, n, mode)
        accumulate(out, lo, hi, up, down)
    return out


def compare(ref: np.ndarray, test: np.ndarray) -> dict:
    """Normalized L1/L2 errors on real and imag parts (accuracy.py:23-64)."""
    out = {}
    for part in ("real", "imag"):
        r = getattr(ref, part).astype(np.float64)
        t = getattr(test, part).astype(np.float64)
        d = r - t
        out[f"l1_{part}"] = float(np.abs(d).sum() / np.abs(r).sum())
        out[f"l2_{part}"] = float(np.sqrt((d * d).sum()) / np.sqrt((r * r).sum()))
    out["pass"] = all(v < 5e-7 for k, v in out.items() if k != "pass")
    return out


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
