# persistent v2: no prefetch (30), prefetch.global.L2 (31), evict-first bulk prefetch (32)
cd $GRAFT_REPO_ROOT
L="timeout 120 python tools/k1_lab.py"
G4RING_V2GEOM=32 timeout 300 python -m pytest tests -x -q -m gpu -k "variant or full_size" 2>&1 | tail -1
for g in 13 30 31 32; do for b in 1 8; do G4RING_V2GEOM=$g $L --batch $b --tag "geom $g"; done; done
