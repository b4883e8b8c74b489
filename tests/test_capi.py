"""The C-ABI library: builds, loads without a GPU, exports every symbol that
include/g4ring.h declares, and its host-only entry points match the reference.
No compute calls (CPU-only container)."""
import ctypes
import json
import re

import pytest

from paper_2105_00027_b200 import _lib
from paper_2105_00027_b200 import errors
from paper_2105_00027_b200 import tensor as T

from .conftest import GOLDEN, ROOT


def header_symbols():
    text = (ROOT / "include" / "g4ring.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(g4_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load(build_if_missing=True)
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table out of sync with include/g4ring.h"
    assert lib.g4_abi_version() == _lib.ABI_VERSION


def test_payload_bytes():
    lib = _lib.load()
    assert lib.g4_payload_bytes(512, _lib.G4_C128) == 2 * 552 * 584 * 16
    assert lib.g4_payload_bytes(4608, _lib.G4_C64) == 2 * 4648 * 4681 * 8  # odd pitch for complex64
    assert lib.g4_payload_bytes(0, _lib.G4_C128) == -1


def test_index_diff_known_answers():
    misc = json.loads((GOLDEN / "misc.json").read_text())
    for a, b, n, want in misc["index_diff"]:
        # any (n_k, n_w) factorisation; the reference works on the combined index
        assert T.index_diff(a, b, T.CombinedIndexSpace(1, n)) == want
    sp = T.CombinedIndexSpace(2, 2)
    for a, b in ((4, 0), (0, -1)):
        with pytest.raises(errors.ContractViolation):
            T.index_diff(a, b, sp)


def test_partition_known_answers():
    misc = json.loads((GOLDEN / "misc.json").read_text())
    for n, p, ranges in misc["partition"]:
        assert [list(r) for r in T.make_partition(n, p).ranges] == ranges
    with pytest.raises(errors.ContractViolation):
        T.make_partition(4, 5)
    with pytest.raises(errors.ContractViolation):
        T.make_partition(4, 0)


@pytest.mark.parametrize("n,p", [(1, 1), (7, 3), (64, 64), (4608, 8), (576, 7)])
def test_partition_invariants(n, p):
    r = T.make_partition(n, p).ranges
    sizes = [hi - lo for lo, hi in r]
    assert r[0][0] == 0 and r[-1][1] == n and max(sizes) - min(sizes) <= 1
    assert all(a[1] == b[0] for a, b in zip(r, r[1:]))


def test_index_space_rejects_bad_dims():
    with pytest.raises(errors.ContractViolation):
        T.CombinedIndexSpace(0, 3)
    sp = T.CombinedIndexSpace(16, 32)
    assert sp.size == 512 and sp.combined(3, 2) == 35


def test_no_cpu_fallback():
    """Slices and payloads refuse host tensors instead of computing on CPU."""
    import torch
    sp = T.CombinedIndexSpace(2, 2)
    with pytest.raises(errors.ContractViolation):
        T.GtSlice(sp, 0, 4, torch.zeros((4, 4, 4), dtype=torch.complex128))


def test_status_mapping():
    lib = _lib.load()
    out = ctypes.c_int64()
    st = lib.g4_index_diff(9, 0, 4, ctypes.byref(out))
    with pytest.raises(errors.ContractViolation, match="out of range"):
        _lib.check(st)


def test_k1_config_host_query():
    """g4_k1_config (host only): the launch g4_accumulate_staged picks per shape."""
    lib = _lib.load()

    def cfg(n, planes, dtype=_lib.G4_C128, nbatch=8):
        out = (ctypes.c_int32 * 9)()
        _lib.check(lib.g4_k1_config(n, planes, nbatch, dtype, out))
        return list(out)

    assert cfg(512, 64)[:5] == [2, 8, 2, 16, 4]      # 16-plane CTA tile
    assert cfg(512, 8)[:5] == [2, 8, 2, 8, 8]        # 8-plane tile for an 8-GPU share
    assert cfg(512, 2)[0] == 1 and cfg(32, 64)[0] == 1  # v1: < 4 planes or N < 64
    assert cfg(4608, 72, _lib.G4_C128_G64)[0] == 2
    assert cfg(512, 64)[8] == 0                         # exact mode: slice read and written by K1
    _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED))
    try:
        assert cfg(512, 64)[:8] == [3, 8, 4, 16, 16, 4, 1, 16] and cfg(512, 64)[8] == 1  # v3: persistent, TMEM
        assert cfg(512, 64, _lib.G4_C128_G64)[0] == 3                          # mixed payloads: v3 too
        assert cfg(4608, 72)[:6] == [3, 8, 4, 16, 16, 3]                        # N = 4608: geometry 43
        assert cfg(512, 64, _lib.G4_C64)[:5] == [2, 8, 4, 16, 8]               # complex64 slices: geometry 12
        assert cfg(512, 64, nbatch=2)[8] == 0                                  # not for B < 4
        assert cfg(512, 8)[:5] == [2, 8, 2, 8, 8] and cfg(512, 8)[8] == 1      # 8-GPU share: geometry 19, deferred
    finally:
        _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_EXACT))
    with pytest.raises(errors.ContractViolation):
        _lib.check(lib.g4_k1_config(0, 8, 8, _lib.G4_C128, (ctypes.c_int32 * 9)()))
    with pytest.raises(errors.ContractViolation):
        _lib.check(lib.g4_k1_config(512, 8, 8, 7, (ctypes.c_int32 * 9)()))
