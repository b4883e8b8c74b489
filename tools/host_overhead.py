import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2105_00027_b200 import tensor as T, _lib
dev = torch.device("cuda", 0)
for n, planes, B in ((64, 16, 8), (512, 8, 8)):
    sp = T.CombinedIndexSpace(1, n)
    sl = T.GtSlice.zeros(sp, 0, planes, device=dev)
    gs = [T.generate_gsigma(0, T.Origin(0, 0, w, 0, 0), sp, "float", device=dev) for w in range(B)]
    for _ in range(10): T.accumulate_g4_batch(sl, gs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200): T.accumulate_g4_batch(sl, gs)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"n={n} P={planes} B={B}: host {1e6*(t1-t0)/200:.1f} us/call, wall {1e6*(t2-t0)/200:.1f} us/call")
