#!/usr/bin/env python
"""Per-tile timeline of K1 v3 (lab; needs G4RING_V3_TRACE support in the library).

    python tools/v3_trace.py [--batch 8] [--planes 64]

Runs a few fused passes at the bench shape with G4RING_V3_TRACE=<tmp file>,
then summarises, per tile (clock64 cycles, per CTA): consumer tile time, the
epilogue's drain time, and the consumers' wait for a drained TMEM buffer."""
from __future__ import annotations

import argparse
import os
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--planes", type=int, default=64)
    ap.add_argument("--passes", type=int, default=4)
    a = ap.parse_args()
    path = tempfile.mktemp(suffix=".bin")
    os.environ["G4RING_V3_TRACE"] = path
    import numpy as np
    import torch
    from paper_2105_00027_b200 import _lib, tensor as T
    lib = _lib.load()
    _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED))
    dev = torch.device("cuda", 0)
    sp = T.CombinedIndexSpace(16, 32)
    sl = T.GtSlice.zeros(sp, 0, a.planes, device=dev)
    gs = [T.GSigma.empty(sp, device=dev) for _ in range(a.batch)]
    T.fill_gsigmas(gs, 0, [T.Origin(0, 0, w, 0, 0) for w in range(a.batch)], "float")
    for _ in range(a.passes):
        T.accumulate_g4_batch(sl, gs)
    torch.cuda.synchronize()
    raw = np.fromfile(path, dtype=np.int64)
    grid = raw.size // (a.passes * 32 * 8)
    tr = raw.reshape(a.passes, grid, 32, 8)[-1].copy()  # last pass
    tr[:, 31, :] = 0  # row 31: globaltimer stamps (below)
    # [0] epi q0 tfull done, [1] epi q0 drained, [2] cons w0 tile done, [3] cons w0 tready wait,
    # [4] cons w0 tile start, [5] cons w0 fill-wait cycles, [6] epi q3 tfull done, [7] epi q3 drained
    ok = tr[:, :, 4] > 0
    ntile = ok.sum(1)
    start = np.where(ok, tr[:, :, 4], 0)
    t0 = start[:, 0:1]
    def rel(x):
        return np.where(ok, x - t0, 0)
    dur = []
    for c in range(grid):
        k = ntile[c]
        s = tr[c, :k, 4]
        e = tr[c, :k, 2]
        dur += list(e - s)
    dur = np.array(dur)
    drain = np.where(ok, tr[:, :, 1] - tr[:, :, 0], 0)[ok]
    drain3 = np.where(ok, tr[:, :, 7] - tr[:, :, 6], 0)[ok]
    lag = np.where(ok, tr[:, :, 0] - np.maximum(tr[:, :, 2], tr[:, :, 5]), 0)[ok]
    fillw = np.where(ok, tr[:, :, 5], 0)[ok]  # [5]: cycles consumer warp 0 waited for payload fills
    wait = tr[:, :, 3][ok]
    total = (np.max(np.where(ok, tr[:, :, 2], 0), 1) - tr[:, 0, 4])
    pct = lambda x: f"median {np.median(x):8.0f}  p90 {np.percentile(x, 90):8.0f}  max {np.max(x):8.0f}  mean {np.mean(x):8.0f}"
    print(f"grid {grid}, tiles per CTA {ntile.min()}-{ntile.max()}, CTA span (cycles): {pct(total)}")
    print(f"consumer tile (w0 start -> w0 done): {pct(dur)}")
    print(f"w0 fill waits per tile:              {pct(fillw)}")
    print(f"epilogue start lag after w0/w7 done: {pct(lag)}")
    print(f"epilogue drain q0 (tfull -> tready):  {pct(drain)}")
    print(f"epilogue drain q3:                    {pct(drain3)}")
    print(f"consumer w0 tready wait:             {pct(wait)}  (nonzero in {np.mean(wait > 200) * 100:.0f}% of tiles)")
    # drains of tiles in the last 32-column strip (their chunks wrap: the edge path) vs the rest
    n = 512
    nx, ny, nz = -(-a.planes // 16), -(-n // 32), -(-n // 16)

    def tile_y(lin):  # tile_coord (g4_k1.cuh) with TILE_BY = 16, TILE_BZ = 32: the column chunk
        per_row = nx * ny * 32
        br = lin // per_row
        r = lin - br * per_row
        bze = min(32, nz - br * 32)
        per_blk = nx * 16 * bze
        by = r // per_blk
        r -= by * per_blk
        bye = min(16, ny - by * 16)
        r //= nx
        return by * 16 + r % bye
    edge, inner = [], []
    for c in range(grid):
        for k in range(min(ntile[c], 31)):
            d = tr[c, k, 1] - tr[c, k, 0]
            if tr[c, k, 0] == 0 or tr[c, k, 1] == 0:
                continue
            (edge if tile_y(c + k * grid) == ny - 1 else inner).append(d)
    if edge and inner:
        print(f"drain q0, edge-strip tiles ({len(edge)}): {pct(np.array(edge))}")
        print(f"drain q0, interior tiles ({len(inner)}):   {pct(np.array(inner))}")
    g = raw.reshape(a.passes, grid, 32, 8)[-1][:, 31, :5].astype(np.float64)  # globaltimer ns
    t0 = g[:, 0].min()
    us = lambda x: f"median {np.median(x):7.2f}  min {np.min(x):7.2f}  max {np.max(x):7.2f} us"
    print("globaltimer (us from the first CTA entry):")
    print(f"  CTA entry:                 {us((g[:, 0] - t0) / 1e3)}")
    print(f"  first payload landed:      {us((g[:, 1] - g[:, 0]) / 1e3)}  (after its CTA entry)")
    print(f"  consumers done:            {us((g[:, 2] - t0) / 1e3)}")
    print(f"  epilogue done:             {us((g[:, 3] - t0) / 1e3)}")
    print(f"  producer done:             {us((g[:, 4] - t0) / 1e3)}")
    print(f"  kernel span (entry->last done): {(max(g[:, 2].max(), g[:, 3].max()) - t0) / 1e3:.2f} us")
    os.unlink(path)


if __name__ == "__main__":
    main()
