# persistent geometry 13: plain (30), payload evict_last (31), + next-tile G4 L2 prefetch (32)
cd $GRAFT_REPO_ROOT
G4RING_V2GEOM=32 timeout 300 python -m pytest tests -x -q -m gpu -k "variant or full_size or bench_workload" 2>&1 | tail -1
L="timeout 120 python tools/k1_lab.py"
for g in 13 30 31 32; do for b in 1 8 16; do G4RING_V2GEOM=$g $L --batch $b --tag "geom $g"; done; done
for g in 13 32; do G4RING_V2GEOM=$g $L --batch 8 --n 4608 --planes 72 --iters 3 --tag "geom $g c4"; done
