#!/usr/bin/env python
"""Config-4-sized ring near the memory limit of the box: R rank processes on
the available GPU(s), each owning 72 planes of the N = 4608 index space
(config 4's per-GPU share: 24.5 GB of complex128 G4 per rank), one ring of R.
Every walker of every rank travels the ring.  No full gather: the first and
last plane of every rank's slice are checked against the C oracle.

    python tools/ring_capacity.py [--ranks 6] [--measurements 1]

On an 8-GPU node, --ranks 8 is BASELINE config 4 itself: 576 planes, 196 GB of
G4 across the 8 GPUs, one rank per GPU.

Prints one JSON line (total G4 bytes, per-rank bytes, round time, max
relative error of the sampled planes).  Measurement tool, not a test.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2105_00027_b200 import engine as E  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=6)
    ap.add_argument("--measurements", type=int, default=1)
    a = ap.parse_args()
    per = 72
    planes = per * a.ranks
    samples = tuple(sorted({q for r in range(a.ranks) for q in (r * per, r * per + per - 1)}))
    cfg = E.ExperimentConfig(n_k=36, n_w=128, world_size=a.ranks, subring_size=a.ranks, lanes=1,
                             measurements=a.measurements, seed=3, value_mode="float", planes=planes, batch=1,
                             gather=False, sample_planes=samples, timeout_s=600.0, instrument=False)
    t0 = time.monotonic()
    rep = E.run_experiment(cfg)
    wall = time.monotonic() - t0
    n = 4608
    walkers = [O.gsigma(cfg.seed, wr, 0, m, n, "float") for wr in range(a.ranks) for m in range(a.measurements)]
    worst = 0.0
    for k3, got in sorted(rep.samples.items()):
        ref = np.zeros((1, n, n), np.complex128)
        for up, down in walkers:
            O.accumulate(ref, k3, k3 + 1, up, down)
        worst = max(worst, float(np.abs(got - ref[0]).max() / np.abs(ref[0]).max()))
    g4_bytes = planes * n * n * 16
    print(json.dumps({"ranks": a.ranks, "planes": planes, "n": n, "g4_bytes": g4_bytes,
                      "g4_bytes_per_rank": per * n * n * 16, "measurements": a.measurements,
                      "sampled_planes": list(samples), "max_rel_err": worst, "tolerance": 1e-10,
                      "ok": worst < 1e-10, "wall_s": wall,
                      "round_gpu_ms": {str(r): v for r, v in rep.round_ms.items()},
                      "per_rank": [{"rank": r, "slice": list(rep.slices[r]), "peak_device_bytes": rep.memory_peaks[r],
                                    "gpu_ms": rep.round_ms.get(r)} for r in sorted(rep.slices)],
                      "visible_gpus": torch.cuda.device_count(),
                      "config4": planes == 576,
                      "note": ("one rank per GPU" if torch.cuda.device_count() >= a.ranks else
                               "ranks share the box's GPU(s); times are not per-GPU throughput")}),
          flush=True)


if __name__ == "__main__":
    main()
