"""ctypes binding of libg4ring.so (the C ABI declared in include/g4ring.h).

There is no fallback: if the library cannot be loaded, every product entry
point raises.  The library is built in-tree (``python -m
paper_2105_00027_b200.build``) and travels to the GPU box with the repo.
"""
from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from .errors import (ConfigError, ContractViolation, DeadlockError, RingAccError,
                     TransportError)

LIB_PATH = Path(__file__).resolve().parent / "libg4ring.so"

G4_OK, G4_ERR_CONTRACT, G4_ERR_CONFIG, G4_ERR_TRANSPORT, G4_ERR_DEADLOCK, G4_ERR_CUDA = range(6)
G4_C128, G4_C64, G4_C128_G64 = 0, 1, 2
G4_MODE_FLOAT, G4_MODE_INTEGER = 0, 1
G4_CHANNEL_EQ1 = 0
G4_ARITH_EXACT, G4_ARITH_FUSED = 0, 1
G4_MAX_BATCH = 64
G4_IPC_HANDLE_BYTES = 64
G4_HALO_ROWS, G4_HALO_COLS = 40, 72
G4_OP_WORDS = 8
G4_OP_ACC, G4_OP_WAIT, G4_OP_WRITE, G4_OP_COPY, G4_OP_RECORD, G4_OP_WAIT_EVENT, G4_OP_GEN, G4_OP_HALO = range(1, 9)
ABI_VERSION = 1

# (name, restype, argtypes) for every symbol include/g4ring.h declares.
_i32, _i64, _u64, _vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p
_vpp = ctypes.POINTER(ctypes.c_void_p)
_i64p = ctypes.POINTER(ctypes.c_int64)
SIGNATURES = {
    "g4_last_error": (ctypes.c_char_p, []),
    "g4_abi_version": (_i32, []),
    "g4_payload_bytes": (_i64, [_i32, _i32]),
    "g4_staged_dims": (_i32, [_i32, _i32, ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
    "g4_index_diff": (_i32, [_i64, _i64, _i64, _i64p]),
    "g4_make_partition": (_i32, [_i64, _i64, _i64p]),
    "g4_prepare_g": (_i32, [_vpp, _vpp, _vpp, _i32, _i32, _i32, _i32, _vp]),
    "g4_generate": (_i32, [_vpp, _vpp, _vpp, _i32, _u64, _i64p, _i64p, _i64p, _i32, _i32, _i32, _vp]),
    "g4_accumulate_staged": (_i32, [_vp, _i64, _i64, _i32, _vpp, _i32, _i32, _i32, _vp]),
    "g4_set_kernel_variant": (_i32, [_i32]),
    "g4_set_arith_mode": (_i32, [_i32]),
    "g4_get_arith_mode": (_i32, []),
    "g4_last_k1_geometry": (_i32, []),
    "g4_k1_config": (_i32, [_i32, _i64, _i32, _i32, ctypes.POINTER(_i32)]),
    "g4_accumulate_workspace_bytes": (_i64, [_i32, _i32, _i32]),
    "g4_accumulate": (_i32, [_vp, _i64, _i64, _i32, _vpp, _vpp, _i32, _i32, _i32, _vp, _i64, _vp]),
    "g4_ipc_export": (_i32, [_vp, _vp, _i64p]),
    "g4_ipc_import": (_i32, [_vp, _i64, _vpp]),
    "g4_ipc_close": (_i32, [_vp]),
    "g4_copy_async": (_i32, [_vp, _vp, _i64, _vp]),
    "g4_peer_copy_fallbacks": (_i64, []),
    "g4_copy_payload_cores": (_i32, [_vp, _vp, _i32, _i32, _i32, _vp]),
    "g4_fill_halo": (_i32, [_vpp, _i32, _i32, _i32, _vp]),
    "g4_preload_ring_kernels": (_i32, []),
    "g4_flag_write": (_i32, [_vp, _u64, _vp]),
    "g4_flag_wait": (_i32, [_vp, _u64, _vp]),
    "g4_flag_host_wait": (_i32, [_vp, _u64, _i64]),
    "g4_reduce_sum": (_i32, [_vp, _vpp, _i32, _i64, _i32, _vp]),
    "g4_round_program_create": (_i32, [_i64p, _i32, _vpp, _i32, _i64p, _i32, _vpp, _i32, _vpp, _i32, _vp, _i64, _i64,
                                       _i32, _i32, _i32, _u64, _i32, _i64, _i32, _vpp]),
    "g4_round_program_run": (_i32, [_vp, _i64, _i32]),
    "g4_round_program_k1_ms": (_i32, [_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i32)]),
    "g4_round_program_destroy": (_i32, [_vp]),
    "g4_ring_create": (_i32, [_vp, _i32, _vp, _vp, _vpp]),
    "g4_ring_measure": (_i32, [_vp, _i64, _i32]),
    "g4_ring_stage": (_i32, [_vp, _vpp, _vpp, _i32, _i32]),
    "g4_ring_wait": (_i32, [_vp, _i64]),
    "g4_ring_slice": (_i32, [_vp, _vpp, _i64p, _i64p]),
    "g4_ring_reduce": (_i32, [_vp]),
    "g4_ring_destroy": (_i32, [_vp]),
}

G4_GROUP_SUBRING, G4_GROUP_POSITION = 0, 1
# int32_t (*g4_allgather_fn)(void* ctx, int32_t group, const void* send, int64_t bytes, void* recv)
ALLGATHER_FN = ctypes.CFUNCTYPE(_i32, _vp, _i32, _vp, _i64, _vp)


class RingConfig(ctypes.Structure):
    """g4_ring_config (include/g4ring.h)."""

    _fields_ = [("n_k", _i32), ("n_w", _i32), ("world_size", _i32), ("subring_size", _i32), ("lanes", _i32),
                ("alternate", _i32), ("batch", _i32), ("dtype", _i32), ("planes", _i64), ("value_mode", _i32),
                ("reserved", _i32), ("seed", _u64)]

_lock = threading.Lock()
_lib = None


class LibraryUnavailable(RingAccError):
    """libg4ring.so is missing or failed to load (there is no CPU fallback)."""


def load(build_if_missing: bool = False):
    """Load (once) and type the C ABI.  Raises LibraryUnavailable on failure."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists() and build_if_missing:
            from .build import build
            build()
        if not LIB_PATH.exists():
            raise LibraryUnavailable(
                f"{LIB_PATH} not built; run `python -m paper_2105_00027_b200.build`")
        try:
            lib = ctypes.CDLL(str(LIB_PATH))
        except OSError as exc:  # pragma: no cover
            raise LibraryUnavailable(f"cannot load {LIB_PATH}: {exc}") from None
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        if lib.g4_abi_version() != ABI_VERSION:
            raise LibraryUnavailable("libg4ring.so ABI version mismatch")
        _lib = lib
        return lib


def check(status: int, what: str = "") -> None:
    """Map a g4_status onto the reference exception hierarchy (errors.py:8-27)."""
    if status == G4_OK:
        return
    msg = (_lib.g4_last_error() or b"").decode(errors="replace") if _lib else ""
    msg = f"{what}: {msg}" if what else msg
    if status == G4_ERR_CONTRACT:
        raise ContractViolation(msg)
    if status == G4_ERR_CONFIG:
        raise ConfigError(msg)
    if status == G4_ERR_DEADLOCK:
        raise DeadlockError(msg)
    if status == G4_ERR_TRANSPORT:
        raise TransportError(msg)
    raise RuntimeError(f"CUDA error in libg4ring: {msg}")


def ptr_array(ptrs) -> ctypes.Array:
    arr = (ctypes.c_void_p * max(len(ptrs), 1))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def i64_array(vals) -> ctypes.Array:
    arr = (ctypes.c_int64 * max(len(vals), 1))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr
