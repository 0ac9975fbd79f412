"""GPU: the multi-process mode (one process per rank, symmetric heap,
MPIX_World_init_mp) — SURVEY.md §8(f) item 2. Two torchrun processes share
GPU 0 here (the box has one GPU); on an 8-GPU box each gets its own. The
worker (tests/mp_worker.py) checks every payload and result exactly."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(600)
@pytest.mark.parametrize("nproc", [2, 3])
def test_multi_process_world(nproc):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
           str(nproc), "--master-addr", "127.0.0.1", "--master-port", str(29600 + nproc),
           os.path.join(ROOT, "tests", "mp_worker.py")]
    env = dict(os.environ, MPIX_SPIN_TIMEOUT_MS="60000")
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=560, cwd=ROOT, env=env)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-4000:]
    for r in range(nproc):
        assert f"MP OK {r}" in out, out[-4000:]
