import sys; sys.path.insert(0, ".")
import torch
from paper_2105_00027_b200 import tensor as T, _lib
lib = _lib.load(); _lib.check(lib.g4_set_kernel_variant(2))
sp = T.CombinedIndexSpace(1, 96)
sl = T.GtSlice.zeros(sp, 0, 96, device="cuda", dtype=torch.complex64)
gs = [T.generate_gsigma(1, T.Origin(0, 0, w, 0, 0), sp, device="cuda", dtype=torch.complex64) for w in range(2)]
T.accumulate_g4_batch(sl, gs)
torch.cuda.synchronize()
print("ok", sl.data.abs().sum().item())
