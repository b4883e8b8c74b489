"""Drop-in surface checks that need no GPU: reference configs accepted as-is,
the same ConfigError cases as the reference validator, the error hierarchy
caught by the reference's ``except`` clauses, and the wire format byte for
byte.  Runs where the reference package is importable (this build container);
skipped elsewhere (the GPU box has no /root/reference)."""
import os
import subprocess
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np
import pytest

REF_SRC = Path("/root/reference/pkg/src")
if REF_SRC.is_dir() and str(REF_SRC) not in sys.path:
    sys.path.append(str(REF_SRC))
ringacc = pytest.importorskip("ringacc")
from ringacc import config as RC  # noqa: E402
from ringacc import wire as RW  # noqa: E402

from paper_2105_00027_b200 import engine as E  # noqa: E402
from paper_2105_00027_b200 import wire as W  # noqa: E402
from paper_2105_00027_b200.errors import ConfigError  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent


def ref_desk(**kw):
    base = dict(n_k=2, n_w=2, world_size=4, subring_size=2, lanes=1, measurements=2, seed=11,
                value_mode="integer", transport="inprocess", timeout_s=10.0)
    base.update(kw)
    return RC.ExperimentConfig(**base)


def test_reference_config_object_accepted():
    rc = ref_desk(lanes=3, direction="alternate")
    c = E.as_config(rc)
    E.validate_config(rc)
    E.validate_config(c)
    for f in ("n_k", "n_w", "world_size", "subring_size", "lanes", "measurements", "seed", "value_mode",
              "transport", "direction", "timeout_s", "instrument", "out_dir", "link", "sweep", "memory"):
        assert getattr(c, f) == getattr(rc, f), f
    assert c.planes is None and c.batch == 1 and c.dtype == "c128"
    assert c.to_dict()["link"] == rc.link.to_dict()


def test_reference_kwargs_and_positional_construction():
    rc = ref_desk()
    kw = {k: getattr(rc, k) for k in ("n_k", "n_w", "world_size", "subring_size", "lanes", "measurements", "seed",
                                       "value_mode", "transport", "direction", "link", "timeout_s", "instrument",
                                       "out_dir", "sweep", "memory", "ring_steps_override", "fault")}
    c = E.ExperimentConfig(**kw)
    E.validate_config(c)
    pos = E.ExperimentConfig(2, 2, 4, 2, 1, 2, 11, "integer", "inprocess", "forward")
    assert pos.transport == "inprocess" and pos.direction == "forward"


def test_reference_json_config_accepted(tmp_path):
    p = tmp_path / "c.json"
    p.write_text('{"n_k": 4, "n_w": 8, "world_size": 8, "subring_size": 4, "lanes": 2, "measurements": 3,'
                 ' "transport": "sim", "link": {"latency": 1e-6}, "sweep": {"subrings": [1, 2]},'
                 ' "memory": {"entry_bytes": 16}}')
    rc = RC.load_config(p)
    c = E.as_config(rc)
    E.validate_config(c)
    assert c.transport == "sim" and c.sweep.subrings == (1, 2)
    assert E.as_config(rc.to_dict()).to_dict()["link"] == rc.link.to_dict()


BAD = [dict(n_k=0), dict(lanes=1000), dict(world_size=6, subring_size=4), dict(seed=-1),
       dict(value_mode="x"), dict(transport="mpi"), dict(direction="sideways"), dict(timeout_s=0),
       dict(n_k=1, n_w=2, world_size=4, subring_size=1)]


@pytest.mark.parametrize("kw", BAD, ids=[str(b) for b in BAD])
def test_same_config_errors_as_reference(kw):
    rc = ref_desk(**kw)
    with pytest.raises(ringacc.errors.ConfigError):
        RC.validate_config(rc)
    with pytest.raises(ConfigError):
        E.validate_config(rc)
    with pytest.raises(ConfigError):
        E.validate_config(E.as_config(rc))


def test_unknown_dict_key_rejected():
    with pytest.raises(ConfigError):
        E.as_config(dict(n_k=2, n_w=2, world_size=1, subring_size=1, lanes=1, measurements=1, bogus=1))


def test_errors_caught_by_reference_clauses():
    """With ringacc importable, this package's errors derive from ringacc.errors
    (fresh interpreter: the package must import after the reference is on the
    path)."""
    code = ("import ringacc.errors as R\n"
            "from paper_2105_00027_b200 import errors as E\n"
            "assert E.REFERENCE_ERRORS\n"
            "for ours, ref in [(E.ContractViolation, R.ContractViolation), (E.ConfigError, R.ConfigError),\n"
            "                  (E.DeadlockError, R.DeadlockError), (E.TransportError, R.RingAccError)]:\n"
            "    try:\n"
            "        raise ours('x')\n"
            "    except ref:\n"
            "        pass\n"
            "import pickle\n"
            "d = pickle.loads(pickle.dumps(E.DeadlockError('m', rank=1, lane=2, step=3)))\n"
            "assert (d.rank, d.lane, d.step) == (1, 2, 3) and isinstance(d, R.TransportError)\n"
            "print('ok')\n")
    env = dict(os.environ, PYTHONPATH=f"{REF_SRC}:{ROOT}")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr


def test_errors_standalone_without_reference():
    code = ("import sys; sys.modules['ringacc'] = None\n"
            "from paper_2105_00027_b200 import errors as E\n"
            "assert not E.REFERENCE_ERRORS and issubclass(E.DeadlockError, E.RingAccError)\n"
            "print('ok')\n")
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr


@pytest.mark.parametrize("shape", [(3,), (2, 4, 4), (0, 5)])
def test_array_wire_bytes_match_reference(shape):
    rng = np.random.default_rng(1)
    a = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    assert W.serialize_array(a) == RW.serialize_array(a)
    assert np.array_equal(W.deserialize_array(RW.serialize_array(a)), a)
    assert W.GSIGMA_HEADER_BYTES == RW.GSIGMA_HEADER_BYTES


def test_rank_main_dispatch_forms():
    """rank_main(rt, world, cfg) with a communicator takes the comm path;
    rank_main(cfg) the device ring (not run here: no GPU)."""
    assert E._is_config(ref_desk()) and E._is_config(E.as_config(ref_desk()))
    assert not E._is_config(object())
    c = replace(E.as_config(ref_desk()), lanes=2)
    assert c.lanes == 2
