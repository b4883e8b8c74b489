"""A/B of the bench's timed loop for short K1 passes (8-plane slice): per-step
CUDA event pairs vs none, 6 vs 20 steps.  Measurement tool."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2105_00027_b200 import tensor as T  # noqa: E402

dev = torch.device("cuda", 0)
sp = T.CombinedIndexSpace(16, 32)
sl = T.GtSlice.zeros(sp, 0, 8, device=dev)
pools = [[T.GSigma.empty(sp, device=dev) for _ in range(8)] for _ in range(2)]
for i, pool in enumerate(pools):
    T.fill_gsigmas(pool, 0, [T.Origin(0, 0, w, i, 0) for w in range(8)], "float")
st = torch.cuda.current_stream(dev)
for events in (False, True):
    for steps in (6, 20, 100):
        for i in range(5):
            T.accumulate_g4_batch(sl, pools[i % 2])
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        a.record(st)
        for i in range(steps):
            if events:
                ev[i][0].record(st)
            T.accumulate_g4_batch(sl, pools[i % 2])
            if events:
                ev[i][1].record(st)
        b.record(st)
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / steps
        k = sum(x.elapsed_time(y) for x, y in ev) * 1e3 / steps if events else float("nan")
        print(f"events={events} steps={steps}: {us:.1f} us/step, kernel {k:.1f} us", flush=True)
