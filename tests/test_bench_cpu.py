"""bench.py contract parts that run without a GPU: the reference arm's JSON
line (the CPU restatement of accumulate_g4 on the host cores) and the ring
model line the N > 1 bench embeds."""
import json
import subprocess
import sys

from .conftest import ROOT


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "2", "--warmup", "1", "--batch", "4"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"].startswith("c1")


def test_ring_model_line():
    sys.path.insert(0, str(ROOT))
    import bench
    m = bench.ring_model_line(512, 64, 8, 8, "c128", 8, 1)
    assert m["ring_hidden"] is False and m["round_ms"] > m["k1_ms"] > 0
    m4 = bench.ring_model_line(4608, 576, 8, 8, "c128", 8, 1)
    assert m4["ring_hidden"] is True
