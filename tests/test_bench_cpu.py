"""CPU: the bench's multi-process launch path (torchrun, world_size 2, gloo
rendezvous on 127.0.0.1) through the reference arm, which runs on host cores:
rank 0 prints exactly one JSON line with impl "reference", rank 1 prints
nothing and both exit 0 (the contract the driver's scaling run relies on)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_built():
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libstreamix_ref.so"))


@pytest.mark.skipif(not _ref_built(), reason="oracle/_ref not built (run __graft_entry__.build())")
def test_reference_arm_under_torchrun_two_ranks():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "2", "--warmup", "1",
           "--size", str(1 << 20)]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "reference"
