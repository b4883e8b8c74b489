"""A C++ host of the native ring driver (tests/native/ring_threads.cpp): ranks
are threads of one process sharing the GPU, the control plane an in-process
all-gather, no Python on the path.  Compiled with nvcc and linked against
libg4ring.so; its reduced G4 is checked bitwise against the C oracle inside the
program.  Also: ranks spread over every visible GPU (one GPU on the test box:
the same code path with peer access to itself), and host-fed rounds
(g4_ring_stage every round) with rank 0 delayed.  GPU only."""
import subprocess

import pytest

from paper_2105_00027_b200.build import nvcc

from .conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ring_threads(tmp_path_factory):
    exe = tmp_path_factory.mktemp("native") / "ring_threads"
    lib = ROOT / "paper_2105_00027_b200"
    cmd = [nvcc(), "-std=c++17", "-Wno-deprecated-gpu-targets", "-Xcompiler", "-ffp-contract=off",
           "-I", str(ROOT / "include"), str(ROOT / "tests" / "native" / "ring_threads.cpp"),
           str(ROOT / "oracle" / "g4_oracle.c"), "-L", str(lib), "-lg4ring", "-Xlinker", f"-rpath={lib}",
           "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True, timeout=300)
    return exe


@pytest.mark.parametrize("args", [["4", "2", "2", "1", "2", "3"],    # 2 sub-rings of 2, alternate lanes
                                  ["3", "3", "1", "0", "1", "2"],    # one ring of 3
                                  ["2", "1", "2", "0", "2", "2"],    # S = 1: replicas + reduce
                                  ["4", "4", "2", "1", "1", "3", "0"],             # ranks over every visible GPU
                                  ["4", "4", "2", "0", "2", "4", "1", "1", "30"],  # host-fed, rank 0 late
                                  ["3", "3", "1", "0", "1", "3", "0", "1", "15"]])
def test_cpp_host_ring(ring_threads, args):
    out = subprocess.run([str(ring_threads), *args], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "ring_threads ok" in out.stdout
