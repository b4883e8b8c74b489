#!/usr/bin/env python
"""Host cost of one K1 call through the Python API (ctypes, tensor-map cache,
launch) against its device time: if the host took longer than the device, the
bench's back-to-back launches would leave the GPU idle between passes.

    python tools/host_overhead.py      (GPU box)"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2105_00027_b200 import _lib, tensor as T  # noqa: E402

dev = torch.device("cuda", 0)
lib = _lib.load()
_lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED))
for n_k, n_w, planes, B in ((1, 64, 16, 8), (16, 32, 8, 8), (16, 32, 64, 8)):
    sp = T.CombinedIndexSpace(n_k, n_w)
    sl = T.GtSlice.zeros(sp, 0, planes, device=dev)
    pools = [[T.generate_gsigma(0, T.Origin(0, 0, w, i, 0), sp, "float", device=dev) for w in range(B)]
             for i in range(2)]
    for i in range(10):
        T.accumulate_g4_batch(sl, pools[i % 2])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    for i in range(200):
        T.accumulate_g4_batch(sl, pools[i % 2])
    t1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    print(f"N={sp.size} P={planes} B={B}: host {1e6 * (t1 - t0) / 200:.1f} us/call, "
          f"device {1e3 * a.elapsed_time(b) / 200:.1f} us/call", flush=True)
