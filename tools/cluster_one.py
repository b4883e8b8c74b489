"""One K1 pass through the forced geometry (G4RING_V2GEOM), for compute-sanitizer."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2105_00027_b200 import tensor as T  # noqa: E402
n, planes, nb = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (128, 64, 2)))
dev = torch.device("cuda", 0)
sp = T.CombinedIndexSpace(1, n)
sl = T.GtSlice.zeros(sp, 0, planes, device=dev)
gs = [T.generate_gsigma(0, T.Origin(0, 0, w, 0, 0), sp, "integer", device=dev) for w in range(nb)]
T.accumulate_g4_batch(sl, gs)
torch.cuda.synchronize()
print("done", float(sl.data.abs().sum()))
