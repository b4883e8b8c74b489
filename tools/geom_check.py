#!/usr/bin/env python
"""Parity of one forced K1 geometry (G4RING_V2GEOM in the environment) against
the C oracle, exact and fused arithmetic, on small slices and on the bench's
own N = 512 x 64-plane x 8-walker shape:

    G4RING_V2GEOM=25 python tools/geom_check.py [--repeat 3]

Prints one line per case and exits 1 on any mismatch.  Run by
tests/test_gpu_headline.py (production and warp-specialised geometries,
repeated to catch timing-dependent races) and tests/test_gpu_kernels.py
(cluster geometry 22).
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2105_00027_b200 import _lib, tensor as T  # noqa: E402

CASES = [  # n, lo, hi, walkers, payload dtype
    (512, 0, 64, 8, "c128"),
    (256, 3, 67, 5, "c128"),
    (96, 0, 32, 4, "c128"),
    (128, 7, 39, 6, "c64"),
    (160, 0, 64, 8, "mixed"),
    (100, 0, 64, 4, "c128"),  # N % 32 != 0: falls back to the plain geometry
]


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--repeat", type=int, default=1)
    args = ap.parse_args()
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    bad = 0
    for arith in [a for _ in range(args.repeat) for a in ("exact", "fused")]:
        _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED if arith == "fused" else _lib.G4_ARITH_EXACT))
        for n, lo, hi, nb, dt in CASES:
            sp = T.CombinedIndexSpace(1, n)
            sdt = torch.complex64 if dt == "c64" else torch.complex128
            gdt = torch.complex128 if dt == "c128" else torch.complex64
            for mode in ("integer", "float"):
                rng = np.random.default_rng(n + nb)
                start = rng.integers(-3, 4, (hi - lo, n, n)) + 1j * rng.integers(-3, 4, (hi - lo, n, n))
                ref = start.astype(np.complex128)
                sl = T.GtSlice(sp, lo, hi, torch.from_numpy(ref.copy()).to(dev).to(sdt))
                gs = [T.generate_gsigma(4, T.Origin(0, 0, w, 0, 0), sp, mode, device=dev, dtype=gdt)
                      for w in range(nb)]
                T.accumulate_g4_batch(sl, gs)
                torch.cuda.synchronize()
                for g in gs:
                    O.accumulate(ref, lo, hi, g.up.contiguous().cpu().numpy().astype(np.complex128),
                                 g.down.contiguous().cpu().numpy().astype(np.complex128))
                got = sl.data.cpu().numpy().astype(np.complex128)
                err = float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-300))
                tol = 1e-5 if dt == "c64" else (0.0 if (mode == "integer" or arith == "exact") and dt != "mixed"
                                                else 1e-12)
                if dt == "mixed" and mode == "integer":
                    tol = 0.0
                ok = err <= tol
                bad += not ok
                print(f"{arith:5s} n={n} [{lo},{hi}) B={nb} {dt:5s} {mode:7s} max_rel_err={err:.2e} "
                      f"{'ok' if ok else 'MISMATCH'}", flush=True)
    _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_EXACT))
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
