"""Generate tests/golden/models.json from the REAL reference models (run here).

TEST INFRASTRUCTURE ONLY.  Imports ``ringacc.perf`` / ``ringacc.memory`` /
``ringacc.transport.sim`` read-only from /root/reference/pkg/src and records
the closed forms the B200 model re-parameterises:

  perf.py:53-58     message_counts
  perf.py:87-104    slow_link
  perf.py:107-116   predict_elapsed
  perf.py:119-124   model_utilization
  memory.py:26-50   bytes_for_entries / slice_bytes / gsigma_total_bytes
  memory.py:91-115  make_plan

Usage:  PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_models.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "models.json"


def main() -> None:
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF))
    from ringacc.memory import gsigma_total_bytes, make_plan, slice_bytes
    from ringacc.perf import message_counts, model_utilization, predict_elapsed, slow_link
    from ringacc.transport.sim import SimLinkConfig

    links = [SimLinkConfig(), SimLinkConfig(intra_bandwidth=1e6),
             SimLinkConfig(nic_bandwidth=50e9, intra_bandwidth=770e9, latency=8e-6, ranks_per_node=8),
             SimLinkConfig(nic_bandwidth=6e9, latency=1e-3, ranks_per_node=4)]
    perf = []
    for li, link in enumerate(links):
        for s in (1, 2, 3, 4, 6, 8, 12, 16, 24):
            for lanes in (1, 2, 3):
                for msg in (1_000_000, 1_700_000, 8_388_608, 679_477_248):
                    perf.append({"link": li, "s": s, "lanes": lanes, "msg": msg, "n_meas": 10,
                                 "slow": list(slow_link(s, link, lanes)),
                                 "predicted": predict_elapsed(s, 10, msg, link, lanes),
                                 "util": model_utilization(s, link, lanes)})
    counts = {str(s): list(message_counts(s)) for s in (1, 2, 3, 5, 8, 17)}
    plans = []
    for entries, eb, mb, p, k in [(212_336_640, 16, 0.17e9, 3, 7), (512 ** 3, 16, 512 * 512 * 16, 8, 1),
                                  (4608 ** 2 * 576, 16, 4608 * 4608 * 16, 8, 2),
                                  (1024 ** 2 * 64, 8, 1024 * 1024 * 8, 4, 2), (1000, 16, 10.0, 7, 3)]:
        plans.append({"args": [entries, eb, mb, p, k], "plan": make_plan(entries, eb, mb, p, k).to_dict()})
    misc = {"slice_bytes": [[t, p, slice_bytes(t, p)] for t, p in [(1024, 4), (10, 3), (3_397_386_240, 3)]],
            "gsigma_total_bytes": [[m, k, mb, gsigma_total_bytes(m, k, mb)]
                                   for m, k, mb in [("original", 7, 0.17e9), ("distributed", 7, 0.17e9),
                                                    ("distributed", 1, 100.0)]]}
    links_d = [link.to_dict() for link in links]
    OUT.write_text(json.dumps({"links": links_d, "perf": perf, "counts": counts, "plans": plans,
                               "misc": misc}, indent=0))
    print(f"wrote {OUT} ({len(perf)} perf rows, {len(plans)} plans)")


if __name__ == "__main__":
    main()
