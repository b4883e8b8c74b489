"""Generate tests/golden/*.npz from the REAL reference (run in the build container).

TEST INFRASTRUCTURE ONLY.  Imports ``ringacc`` read-only from
/root/reference/pkg/src (which does not exist on the GPU box), runs its own
public functions, and stores their inputs and outputs as small fixtures:

  gen.npz      generate_gsigma (tensor.py:223-228) for several origins/N/modes
  acc.npz      accumulate_g4   (tensor.py:233-251) on random slices/ranges
  c1.npz       BASELINE config 1: N=32 (n_k=4, n_w=8), K3={0}, 16 walkers,
               float seeds 0-4 + integer seed 0
  oracle.npz   oracle_accumulate (tensor.py:276-283) for small ExperimentShapes
  engine.npz   run_experiment (engine.py:323-335) reduced tensors + slice maps
  misc.json    index_diff / make_partition known answers

Usage:  PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def main() -> None:
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF))
    from ringacc.config import ExperimentConfig
    from ringacc.engine import run_experiment
    from ringacc.tensor import (CombinedIndexSpace, ExperimentShape, GtSlice, Origin,
                                accumulate_g4, generate_gsigma, index_diff,
                                make_partition, oracle_accumulate)

    OUT.mkdir(parents=True, exist_ok=True)

    # --- generator ---------------------------------------------------------
    gen = {}
    cases = [(0, (0, 0, 0, 0, 0), 2, 2, "float"), (42, (0, 1, 2, 3, 1), 2, 2, "float"),
             (7, (0, 0, 0, 0, 0), 2, 3, "integer"), (1234, (1, 2, 3, 4, 9), 4, 8, "float"),
             (1234, (1, 2, 3, 4, 9), 4, 8, "integer"), (5, (0, 3, 1, 17, 3), 16, 4, "float"),
             (2**40 + 3, (0, 7, 5, 999, 7), 3, 5, "integer")]
    for i, (seed, o, nk, nw, mode) in enumerate(cases):
        g = generate_gsigma(seed, Origin(*o), CombinedIndexSpace(nk, nw), mode)
        gen[f"c{i}_meta"] = np.array([seed, *o, nk, nw, 0 if mode == "float" else 1], np.uint64)
        gen[f"c{i}_up"], gen[f"c{i}_down"] = g.up, g.down
    np.savez_compressed(OUT / "gen.npz", **gen)

    # --- accumulate on random slices (random nonzero start, random G) --------
    acc = {}
    rng = np.random.default_rng(20260517)
    acc_cases = [(2, 2, 0, 4, 1), (2, 3, 2, 4, 2), (1, 7, 3, 7, 3), (4, 8, 5, 13, 2),
                 (3, 3, 0, 9, 4), (8, 8, 60, 64, 2), (1, 1, 0, 1, 2), (5, 13, 17, 21, 1)]
    for i, (nk, nw, lo, hi, nwalk) in enumerate(acc_cases):
        sp = CombinedIndexSpace(nk, nw)
        n = sp.size
        start = rng.standard_normal((hi - lo, n, n)) + 1j * rng.standard_normal((hi - lo, n, n))
        sl = GtSlice(sp, lo, hi, start.copy())
        ups, downs = [], []
        for w in range(nwalk):
            up = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
            down = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
            from ringacc.tensor import GSigma
            accumulate_g4(sl, GSigma(sp, up, down, Origin(0, 0, w, 0, 0)))
            ups.append(up)
            downs.append(down)
        acc[f"c{i}_meta"] = np.array([nk, nw, lo, hi, nwalk], np.int64)
        acc[f"c{i}_start"], acc[f"c{i}_end"] = start, sl.data
        acc[f"c{i}_up"], acc[f"c{i}_down"] = np.array(ups), np.array(downs)
        acc[f"c{i}_count"] = np.array(sl.meas_count)
    np.savez_compressed(OUT / "acc.npz", **acc)

    # --- BASELINE config 1 ------------------------------------------------------
    c1 = {}
    sp = CombinedIndexSpace(4, 8)
    for seed, mode in [(0, "float"), (1, "float"), (2, "float"), (3, "float"), (4, "float"),
                       (0, "integer")]:
        sl = GtSlice.zeros(sp, 0, 1)
        for w in range(16):
            accumulate_g4(sl, generate_gsigma(seed, Origin(0, 0, w, 0, 0), sp, mode))
        c1[f"{mode}_{seed}"] = sl.data
    np.savez_compressed(OUT / "c1.npz", **c1)

    # --- serial oracle ----------------------------------------------------------
    orc = {}
    for i, (seed, shp, nk, nw, mode) in enumerate([
            (5, (2, 2, 2, 2), 2, 2, "float"), (11, (1, 3, 2, 1), 2, 3, "integer"),
            (2024, (2, 3, 1, 2), 2, 3, "float"), (9, (3, 1, 2, 2), 1, 4, "integer")]):
        out = oracle_accumulate(seed, ExperimentShape(*shp), CombinedIndexSpace(nk, nw), mode)
        orc[f"c{i}_meta"] = np.array([seed, *shp, nk, nw, 0 if mode == "float" else 1], np.int64)
        orc[f"c{i}_tensor"] = out.data
    np.savez_compressed(OUT / "oracle.npz", **orc)

    # --- engine (ring) ------------------------------------------------------------
    eng = {}
    eng_cases = [dict(n_k=2, n_w=2, world_size=4, subring_size=4, lanes=1, measurements=3),
                 dict(n_k=2, n_w=3, world_size=6, subring_size=2, lanes=1, measurements=2),
                 dict(n_k=2, n_w=3, world_size=6, subring_size=3, lanes=2, measurements=2),
                 dict(n_k=2, n_w=4, world_size=4, subring_size=2, lanes=3, measurements=2)]
    for i, kw in enumerate(eng_cases):
        for mode in ("integer", "float"):
            cfg = ExperimentConfig(**kw, seed=77, value_mode=mode, timeout_s=30.0)
            rep = run_experiment(cfg)
            eng[f"c{i}_{mode}_tensor"] = rep.tensor
            eng[f"c{i}_{mode}_meas"] = np.array([rep.meas_counts[r] for r in range(kw["world_size"])])
            eng[f"c{i}_{mode}_slices"] = np.array([rep.slices[r] for r in range(kw["world_size"])])
        eng[f"c{i}_cfg"] = np.array([kw[k] for k in ("n_k", "n_w", "world_size", "subring_size",
                                                     "lanes", "measurements")] + [77], np.int64)
    np.savez_compressed(OUT / "engine.npz", **eng)

    # --- index / partition known answers ---------------------------------------
    misc = {"index_diff": [], "partition": []}
    for (a, b, nk, nw) in [(5, 2, 2, 4), (1, 3, 2, 4), (0, 0, 3, 3), (8, 0, 3, 3),
                           (0, 8, 3, 3), (4607, 0, 36, 128), (0, 4607, 36, 128)]:
        misc["index_diff"].append([a, b, nk * nw, index_diff(a, b, CombinedIndexSpace(nk, nw))])
    for n, p in [(8, 4), (7, 2), (5, 5), (64, 8), (64, 3), (576, 8), (4608, 7), (1, 1)]:
        misc["partition"].append([n, p, [list(r) for r in make_partition(n, p).ranges]])
    (OUT / "misc.json").write_text(json.dumps(misc, indent=1))
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
