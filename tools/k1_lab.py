#!/usr/bin/env python
"""K1 measurement lab: time one configuration of the slice update with CUDA events.

    python tools/k1_lab.py [--n 512] [--planes 64] [--batch 8] [--dtype c128|c64|mixed]
                           [--arith exact|fused] [--iters 20] [--tag TEXT]

Kernel choices come from the library's env knobs (G4RING_KERNEL, G4RING_V2GEOM,
G4RING_EXP), so run one process per variant.  Prints one line:
tag, updates/s, algorithmic GB/s, us per pass.
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2105_00027_b200 import _lib, tensor as T  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--planes", type=int, default=64)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--dtype", default="c128", choices=["c128", "c64", "mixed"])
    ap.add_argument("--arith", default="exact", choices=["exact", "fused"])
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    lib = _lib.load()
    _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED if a.arith == "fused" else _lib.G4_ARITH_EXACT))
    dev = torch.device("cuda", 0)
    n = a.n
    sp = T.CombinedIndexSpace(n, 1)
    gdt = torch.complex128 if a.dtype == "c128" else torch.complex64
    sdt = torch.complex64 if a.dtype == "c64" else torch.complex128
    sl = T.GtSlice.zeros(sp, 0, a.planes, device=dev, dtype=sdt)
    gs = [T.generate_gsigma(0, T.Origin(0, 0, w, 0, 0), sp, "float", device=dev, dtype=gdt)
          for w in range(a.batch)]
    for _ in range(3):
        T.accumulate_g4_batch(sl, gs)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(a.iters):
        T.accumulate_g4_batch(sl, gs)
    ev1.record()
    torch.cuda.synchronize()
    us = ev0.elapsed_time(ev1) * 1e3 / a.iters
    eb = 16 if sdt == torch.complex128 else 8
    pb = 16 if gdt == torch.complex128 else 8
    upd = a.batch * a.planes * n * n
    byt = 2 * a.planes * n * n * eb + a.batch * 2 * n * n * pb
    print(f"{a.tag:28s} n={n} P={a.planes} B={a.batch} {a.dtype}/{a.arith}: "
          f"{upd / us * 1e6:.3e} upd/s  {byt / us * 1e-3:7.0f} GB/s  {us:8.1f} us/pass", flush=True)


if __name__ == "__main__":
    main()
