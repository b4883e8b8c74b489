"""Debug helper: the skip-send deadlock negative control under torchrun, with
stack dumps of every rank after 25 s (faulthandler)."""
import faulthandler
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
faulthandler.dump_traceback_later(25, exit=True)
import torch.distributed as dist  # noqa: E402
from paper_2105_00027_b200 import engine as E  # noqa: E402

dist.init_process_group("gloo")

c = E.ExperimentConfig(n_k=2, n_w=4, world_size=2, subring_size=2, lanes=1, measurements=1, seed=11,
                       value_mode="integer", timeout_s=3.0, fault="skip-send")
try:
    E.rank_main(c)
    print("finished without error", flush=True)
except Exception as exc:
    print("raised", type(exc).__name__, exc, flush=True)
