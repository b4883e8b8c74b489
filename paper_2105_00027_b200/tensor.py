"""Operator API of the hot path -- a drop-in mirror of ``ringacc.tensor``
(/root/reference/pkg/src/ringacc/tensor.py) whose arrays live in B200 HBM.

Same names, argument meaning and errors as the reference:

=====================  ====================================  =========================
reference (tensor.py)  here                                  computed by
=====================  ====================================  =========================
CombinedIndexSpace     CombinedIndexSpace        (31-47)     host
index_diff             index_diff                (50-55)     C ABI g4_index_diff
Origin                 Origin                    (58-74)     host
GSigma                 GSigma                    (77-96)     staged device payload
GtSlice                GtSlice                   (99-136)    device tensor, same layout
make_partition         make_partition            (148-164)   C ABI g4_make_partition
fill_gsigma            fill_gsigma               (215-220)   K3 kernel (g4_generate)
generate_gsigma        generate_gsigma           (223-228)   K3 kernel
accumulate_g4          accumulate_g4             (233-251)   K1 kernel (g4_accumulate_staged)
(batched)              accumulate_g4_batch                   K1, B walkers per HBM pass
ExperimentShape        ExperimentShape           (256-273)   host
oracle_accumulate      oracle_accumulate         (276-283)   K3 + K1 in canonical order
=====================  ====================================  =========================

Differences, all deliberate:
* ``GtSlice.data`` is a CUDA ``torch.Tensor`` (complex128, or complex64) with the
  reference's exact layout ``data[k3 - lo, k1, k2]``.
* ``GSigma`` stores one device tensor ``staged`` of shape (2, N + 40, LD), LD = N + 72
  (odd for complex64):
  spin-planar transposes with a cyclic halo, ``staged[s, r, c] = M_s[c % N, r % N]``
  (``M_0 = up``, ``M_1 = down``) -- the layout the update kernel reads
  row-contiguously (and with TMA boxes) and the form that travels around the ring.  ``g.up`` and
  ``g.down`` are (transposed, zero-copy) views with the reference's meaning.
* There is no CPU path: host arrays passed in are copied to the device; a
  missing CUDA library raises ``LibraryUnavailable``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ContractViolation

ENTRY_BYTES = 16  # complex128 (tensor.py:23)
VALUE_MODES = ("float", "integer")
_MODE_CODE = {"float": _lib.G4_MODE_FLOAT, "integer": _lib.G4_MODE_INTEGER}
_DTYPE_CODE = {torch.complex128: _lib.G4_C128, torch.complex64: _lib.G4_C64}


def staged_shape(n: int, dtype: torch.dtype = torch.complex128) -> tuple[int, int, int]:
    """Shape of one staged payload (include/g4ring.h): (2, ROWS, LD) from g4_staged_dims."""
    lib = _lib.load()
    rows, ld = ctypes.c_int32(), ctypes.c_int32()
    _lib.check(lib.g4_staged_dims(n, _dtype_code(dtype), ctypes.byref(rows), ctypes.byref(ld)), "staged_dims")
    return (2, rows.value, ld.value)


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _require_cuda(t: torch.Tensor, what: str) -> None:
    if not t.is_cuda:
        raise ContractViolation(f"{what} must be a CUDA tensor (this library has no CPU path)")


def _dtype_code(dt: torch.dtype) -> int:
    try:
        return _DTYPE_CODE[dt]
    except KeyError:
        raise ContractViolation(f"unsupported dtype {dt}; use complex128 or complex64") from None


@dataclass(frozen=True)
class CombinedIndexSpace:
    """Discrete index group: ``size = n_k * n_w`` (tensor.py:31-47).  Under the
    convention ``K = w * n_k + k`` (momentum fastest) the first ``n_k * n_wex``
    indices are "all momenta x the first n_wex frequencies"."""

    n_k: int
    n_w: int

    def __post_init__(self):
        if self.n_k < 1 or self.n_w < 1:
            raise ContractViolation(f"index space dims must be >= 1, got ({self.n_k}, {self.n_w})")

    @property
    def size(self) -> int:
        return self.n_k * self.n_w

    def diff(self, a: int, b: int) -> int:
        return index_diff(a, b, self)

    def combined(self, k: int, w: int) -> int:
        """Combined index of momentum k, frequency w (``K = w * n_k + k``)."""
        if not (0 <= k < self.n_k and 0 <= w < self.n_w):
            raise ContractViolation(f"(k, w) = ({k}, {w}) outside ({self.n_k}, {self.n_w})")
        return w * self.n_k + k


def index_diff(a: int, b: int, space: CombinedIndexSpace) -> int:
    """Cyclic K difference ``(a - b) mod N`` (tensor.py:50-55)."""
    lib = _lib.load()
    out = ctypes.c_int64(0)
    _lib.check(lib.g4_index_diff(a, b, space.size, ctypes.byref(out)), "index_diff")
    return int(out.value)


@dataclass(frozen=True)
class Origin:
    """Provenance of one payload (tensor.py:58-74); ``world_rank`` keys the
    generator so content does not depend on sub-ring grouping."""

    subring: int
    rank: int
    lane: int
    meas: int
    world_rank: int

    def sort_key(self):
        return (self.subring, self.rank, self.lane, self.meas)


class GSigma:
    """One walker's payload: spin-up and spin-down N x N matrices (tensor.py:77-96),
    stored staged on the device."""

    def __init__(self, space: CombinedIndexSpace, up=None, down=None, origin: Origin | None = None,
                 *, staged: torch.Tensor | None = None, device=None, dtype=torch.complex128):
        self.space = space
        self.origin = origin or Origin(0, 0, 0, 0, 0)
        n = space.size
        if staged is not None:
            _require_cuda(staged, "GSigma.staged")
            if tuple(staged.shape) != staged_shape(n, staged.dtype) or not staged.is_contiguous():
                raise ContractViolation(f"staged payload must be contiguous {staged_shape(n, staged.dtype)}")
            _dtype_code(staged.dtype)
            self.staged = staged
            return
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.staged = torch.empty(staged_shape(n, dtype), dtype=dtype, device=dev)
        if up is None and down is None:
            self.staged.zero_()
            return
        self.set(up, down)

    # -- reference-meaning accessors (zero-copy views) --------------------------
    @property
    def up(self) -> torch.Tensor:
        n = self.space.size
        return self.staged[0, :n, :n].transpose(0, 1)

    @property
    def down(self) -> torch.Tensor:
        n = self.space.size
        return self.staged[1, :n, :n].transpose(0, 1)

    @property
    def dtype(self) -> torch.dtype:
        return self.staged.dtype

    @property
    def nbytes(self) -> int:
        """Reference payload size (tensor.py:86-89): two N x N matrices."""
        return 2 * self.space.size ** 2 * self.staged.element_size()

    @property
    def device_nbytes(self) -> int:
        """Bytes of the staged device payload (core + halo)."""
        return self.staged.numel() * self.staged.element_size()

    def set(self, up, down) -> None:
        """Stage reference-layout matrices (numpy or torch, host or device) with K2."""
        n = self.space.size
        dev = self.staged.device
        tu = _as_device(up, dev, n)
        td = _as_device(down, dev, n)
        if tu.dtype != td.dtype:
            raise ContractViolation("up and down must share a dtype")
        lib = _lib.load()
        _lib.check(lib.g4_prepare_g(_lib.ptr_array([self.staged.data_ptr()]),
                                    _lib.ptr_array([tu.data_ptr()]), _lib.ptr_array([td.data_ptr()]),
                                    1, n, _dtype_code(tu.dtype), _dtype_code(self.staged.dtype),
                                    _stream_ptr(dev)), "prepare_g")
        # keep the sources alive until the stream has consumed them
        tu.record_stream(torch.cuda.current_stream(dev))
        td.record_stream(torch.cuda.current_stream(dev))

    @classmethod
    def empty(cls, space: CombinedIndexSpace, origin: Origin | None = None, *, device=None,
              dtype=torch.complex128) -> "GSigma":
        return cls(space, None, None, origin, device=device, dtype=dtype)


def _as_device(x, dev: torch.device, n: int) -> torch.Tensor:
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if not isinstance(x, torch.Tensor):
        raise ContractViolation(f"expected an array, got {type(x).__name__}")
    if tuple(x.shape) != (n, n):
        raise ContractViolation(f"matrix shape {tuple(x.shape)} != ({n}, {n})")
    if x.dtype not in _DTYPE_CODE:
        x = x.to(torch.complex128)
    return x.to(dev, non_blocking=True).contiguous()


class GtSlice:
    """Contiguous block of G4 along K3 (tensor.py:99-136):
    ``data[j, k1, k2] = G4(k1, k2, lo + j)``, a CUDA tensor."""

    def __init__(self, space: CombinedIndexSpace, lo: int, hi: int, data: torch.Tensor,
                 meas_count: int = 0):
        n = space.size
        if not (0 <= lo < hi <= n):
            raise ContractViolation(f"invalid axis range [{lo}, {hi}) for N={n}")
        _require_cuda(data, "GtSlice.data")
        if tuple(data.shape) != (hi - lo, n, n) or not data.is_contiguous():
            raise ContractViolation(f"slice data must be contiguous ({hi - lo}, {n}, {n})")
        _dtype_code(data.dtype)
        self.space, self.lo, self.hi, self.data, self.meas_count = space, lo, hi, data, meas_count

    @property
    def entries(self) -> int:
        return (self.hi - self.lo) * self.space.size ** 2

    @property
    def nbytes(self) -> int:
        return self.entries * self.data.element_size()

    @property
    def is_full(self) -> bool:
        return self.lo == 0 and self.hi == self.space.size

    @classmethod
    def zeros(cls, space: CombinedIndexSpace, lo: int, hi: int, *, device=None,
              dtype=torch.complex128) -> "GtSlice":
        n = space.size
        if not (0 <= lo < hi <= n):
            raise ContractViolation(f"invalid axis range [{lo}, {hi}) for N={n}")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        return cls(space, lo, hi, torch.zeros((hi - lo, n, n), dtype=dtype, device=dev))

    @classmethod
    def zeros_full(cls, space: CombinedIndexSpace, **kw) -> "GtSlice":
        return cls.zeros(space, 0, space.size, **kw)


@dataclass(frozen=True)
class PartitionPlan:
    n: int
    p: int
    ranges: tuple[tuple[int, int], ...]


def make_partition(n: int, p: int) -> PartitionPlan:
    """Balanced contiguous split of [0, n) over p ranks (tensor.py:148-164)."""
    lib = _lib.load()
    buf = (ctypes.c_int64 * (2 * max(p, 1)))()
    _lib.check(lib.g4_make_partition(n, p, buf), "make_partition")
    return PartitionPlan(n, p, tuple((buf[2 * i], buf[2 * i + 1]) for i in range(p)))


# -- K3: device generator -------------------------------------------------------

def fill_gsigmas(gs: list[GSigma], seed: int, origins: list[Origin], mode: str = "float") -> None:
    """Regenerate several payloads in place with one K3 launch (no allocation)."""
    if mode not in _MODE_CODE:
        raise ContractViolation(f"unknown value mode {mode!r}")
    if not gs:
        return
    n = gs[0].space.size
    dev = gs[0].staged.device
    dt = gs[0].staged.dtype
    for g in gs:
        if g.space.size != n or g.staged.dtype != dt or g.staged.device != dev:
            raise ContractViolation("fill_gsigmas: payloads must share space, dtype and device")
    lib = _lib.load()
    _lib.check(lib.g4_generate(
        _lib.ptr_array([g.staged.data_ptr() for g in gs]), None, None, len(gs),
        seed & 0xFFFFFFFFFFFFFFFF,
        _lib.i64_array([o.world_rank for o in origins]), _lib.i64_array([o.lane for o in origins]),
        _lib.i64_array([o.meas for o in origins]), n, _MODE_CODE[mode], _dtype_code(dt),
        _stream_ptr(dev)), "generate")
    for g, o in zip(gs, origins):
        g.origin = o


def fill_gsigma(g: GSigma, seed: int, origin: Origin, mode: str = "float") -> None:
    """Regenerate a payload in place (tensor.py:215-220)."""
    fill_gsigmas([g], seed, [origin], mode)


def generate_gsigma(seed: int, origin: Origin, space: CombinedIndexSpace, mode: str = "float", *,
                    device=None, dtype=torch.complex128) -> GSigma:
    """Deterministic payload (tensor.py:223-228); integer mode is bitwise equal
    to the reference, float mode within 2 ulp (device sin/cos)."""
    g = GSigma.empty(space, origin, device=device, dtype=dtype)
    fill_gsigma(g, seed, origin, mode)
    return g


def generate_reference_layout(seed: int, origin: Origin, space: CombinedIndexSpace,
                              mode: str = "float", *, device=None,
                              dtype=torch.complex128) -> tuple[torch.Tensor, torch.Tensor]:
    """K3 writing reference-layout (up, down) matrices (e.g. to ship to a host)."""
    n = space.size
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    up = torch.empty((n, n), dtype=dtype, device=dev)
    down = torch.empty((n, n), dtype=dtype, device=dev)
    lib = _lib.load()
    _lib.check(lib.g4_generate(None, _lib.ptr_array([up.data_ptr()]), _lib.ptr_array([down.data_ptr()]),
                               1, seed & 0xFFFFFFFFFFFFFFFF, _lib.i64_array([origin.world_rank]),
                               _lib.i64_array([origin.lane]), _lib.i64_array([origin.meas]), n,
                               _MODE_CODE[mode], _dtype_code(dtype), _stream_ptr(dev)), "generate")
    return up, down


# -- K1: the update -------------------------------------------------------------

def accumulate_g4_batch(slice_: GtSlice, gs: list[GSigma]) -> None:
    """Apply several payloads to the owned planes in one HBM pass of the slice.
    Bitwise identical to calling ``accumulate_g4`` on each payload in order."""
    if not gs:
        return
    pdt = gs[0].staged.dtype
    for g in gs:
        if g.space != slice_.space:
            raise ContractViolation(f"space mismatch: slice {slice_.space} vs payload {g.space}")
        if g.staged.dtype != pdt:
            raise ContractViolation("all payloads of a batch must share a dtype")
        if g.staged.device != slice_.data.device:
            raise ContractViolation("payload and slice live on different devices")
    code = accumulate_dtype_code(slice_.data.dtype, pdt)
    lib = _lib.load()
    dev = slice_.data.device
    _lib.check(lib.g4_accumulate_staged(
        slice_.data.data_ptr(), slice_.lo, slice_.hi, slice_.space.size,
        _lib.ptr_array([g.staged.data_ptr() for g in gs]), len(gs), code,
        _lib.G4_CHANNEL_EQ1, _stream_ptr(dev)), "accumulate_g4")
    slice_.meas_count += len(gs)


def accumulate_dtype_code(slice_dtype: torch.dtype, payload_dtype: torch.dtype) -> int:
    """C-ABI dtype of an update: same precision, or the mixed complex128 slice /
    complex64 payload mode (G4_C128_G64)."""
    if slice_dtype == payload_dtype:
        return _dtype_code(slice_dtype)
    if slice_dtype == torch.complex128 and payload_dtype == torch.complex64:
        return _lib.G4_C128_G64
    raise ContractViolation(f"payload dtype {payload_dtype} cannot update a {slice_dtype} slice")


def accumulate_g4(slice_: GtSlice, g: GSigma) -> None:
    """Apply one measurement to the K3 planes owned by ``slice_`` (tensor.py:233-251):
    ``G4(K1, K2, K3) += sum_sigma G_sigma(K3-K2, K3-K1) * G_-sigma(K2, K1)``;
    entries outside [lo, hi) are untouched; ``meas_count`` increments by 1."""
    accumulate_g4_batch(slice_, [g])


# -- serial ground truth in canonical order ------------------------------------

@dataclass(frozen=True)
class ExperimentShape:
    """Every (subring, rank, lane, meas) of a run (tensor.py:256-273)."""

    subrings: int
    subring_size: int
    lanes: int
    measurements: int

    def origins(self) -> list[Origin]:
        out = [Origin(s, r, t, m, s * self.subring_size + r)
               for s in range(self.subrings) for r in range(self.subring_size)
               for t in range(self.lanes) for m in range(self.measurements)]
        out.sort(key=Origin.sort_key)
        return out


def oracle_accumulate(seed: int, shape: ExperimentShape, space: CombinedIndexSpace,
                      mode: str = "float", *, device=None, batch: int = 16) -> GtSlice:
    """Serial ground truth (tensor.py:276-283) computed on the device: every
    payload regenerated and applied to a full tensor in canonical origin order."""
    full = GtSlice.zeros_full(space, device=device)
    origins = shape.origins()
    bufs = [GSigma.empty(space, device=full.data.device) for _ in range(min(batch, max(len(origins), 1)))]
    for i in range(0, len(origins), batch):
        chunk = origins[i:i + batch]
        fill_gsigmas(bufs[:len(chunk)], seed, chunk, mode)
        accumulate_g4_batch(full, bufs[:len(chunk)])
    return full
