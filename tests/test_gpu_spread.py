"""GPU: the cross-GPU paths in the single-process World model, ranks spread
over every visible GPU (rank r on GPU r % device_count) so peers reach each
other over NVLink / NVSwitch with system-scope primitives — the reference's
rank -> rank channel write (proj/src/proc_p2p.cpp:47-49) becomes a peer HBM
access. Skipped unless at least two GPUs are visible; on such a box they run
with the rest of the suite, so NVLink parity is checked the moment a
multi-GPU box is used.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2208_13707_b200 import mpix
from tests.gpu_util import gpu_world, sync_all

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 visible GPUs")]


def dev_of(r):
    return r % torch.cuda.device_count()


@pytest.mark.parametrize("n", [0, 8, 4096, 65537, 1 << 20, (16 << 20) + 5])
def test_spread_pairs_isend_irecv_and_blocking(n):
    """Every ordered pair of 4 ranks on distinct GPUs: Isend/Irecv +
    Waitall_enqueue, then blocking Send/Recv_enqueue head to head (eager /
    staged); bytes exact."""
    P = 4
    with gpu_world(P, spread=True) as (w, ctx):
        src = {r: torch.randint(0, 256, (max(n, 1),), dtype=torch.uint8, device=dev_of(r)) for r in range(P)}
        dst = {(r, q): torch.zeros(max(n, 1), dtype=torch.uint8, device=dev_of(r))
               for r in range(P) for q in range(P) if q != r}
        blk = {r: torch.zeros(max(n, 1), dtype=torch.uint8, device=dev_of(r)) for r in range(P)}
        for d in range(torch.cuda.device_count()):
            torch.cuda.synchronize(d)

        def body(r):
            c = ctx[r].comm
            reqs = []
            for q in range(P):
                if q != r:
                    reqs.append(c.irecv_enqueue(dst[(r, q)], n, mpix.MPI_BYTE, q, 5))
            for q in range(P):
                if q != r:
                    reqs.append(c.isend_enqueue(src[r], n, mpix.MPI_BYTE, q, 5))
            mpix.waitall_enqueue(reqs)
            peer = r ^ 1
            c.send_enqueue(src[r], n, mpix.MPI_BYTE, peer, 6)
            c.recv_enqueue(blk[r], n, mpix.MPI_BYTE, peer, 6)

        w.run_ranks(body)
        sync_all(ctx)
        for (r, q), t in dst.items():
            assert torch.equal(t[:n].cpu(), src[q][:n].cpu()), (r, q)
        for r in range(P):
            assert torch.equal(blk[r][:n].cpu(), src[r ^ 1][:n].cpu())


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("count", [1000, 1 << 16, (4 << 20) + 3])
def test_spread_allreduce_bit_exact(P, count):
    """Allreduce_enqueue across GPUs (one-shot fused below 64 KiB, two-shot
    above): bit-exact with the rank-ordered fold."""
    with gpu_world(P, spread=True) as (w, ctx):
        ins = [np.random.default_rng(P * 100 + r).uniform(-1, 1, count).astype(np.float32) for r in range(P)]
        sb = [torch.from_numpy(ins[r]).to(dev_of(r)) for r in range(P)]
        rb = [torch.zeros(count, dtype=torch.float32, device=dev_of(r)) for r in range(P)]
        w.run_ranks(lambda r: ctx[r].comm.allreduce_enqueue(sb[r], rb[r], count, mpix.MPI_FLOAT))
        sync_all(ctx)
        exp = O.allreduce(ins, "f32")
        for r in range(P):
            assert np.array_equal(rb[r].cpu().numpy().view(np.uint32), exp.view(np.uint32)), r


def test_spread_halo_matches_global_oracle():
    from paper_2208_13707_b200.workloads import HaloStencil, coords
    from tests.test_gpu_workloads import global_step
    P, n = 8, 12
    N = 2 * n
    g = np.random.default_rng(3).uniform(-1, 1, (N, N, N)).astype(np.float32)
    with gpu_world(P, spread=True) as (w, ctx):
        blocks = []
        for r in range(P):
            b = HaloStencil(r, n, ctx[r].stream, ctx[r].comm, device=dev_of(r))
            cx, cy, cz = coords(r)
            pad = np.zeros((n + 2, n + 2, n + 2), dtype=np.float32)
            pad[1:-1, 1:-1, 1:-1] = g[cz * n:(cz + 1) * n, cy * n:(cy + 1) * n, cx * n:(cx + 1) * n]
            b.u.copy_(torch.from_numpy(pad.reshape(-1)).to(dev_of(r)))
            blocks.append(b)
        for d in range(torch.cuda.device_count()):
            torch.cuda.synchronize(d)
        w.run_ranks(lambda r: [blocks[r].step() for _ in range(2)])
        sync_all(ctx)
        exp = g
        for _ in range(2):
            exp = global_step(exp, HaloStencil.W0, HaloStencil.W1)
        got = np.zeros_like(g)
        for r in range(P):
            cx, cy, cz = coords(r)
            got[cz * n:(cz + 1) * n, cy * n:(cy + 1) * n, cx * n:(cx + 1) * n] = \
                blocks[r].u.cpu().numpy().reshape(n + 2, n + 2, n + 2)[1:-1, 1:-1, 1:-1]
        assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))
