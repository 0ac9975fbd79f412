"""GPU tests of staged blocking sends (eager completion without the receiver,
proj/src/proc_p2p.cpp:60-62; Appendix A1 of SURVEY.md).

A blocking Send_enqueue larger than the eager slot whose receive is not yet
posted copies the payload into a staging buffer and completes. Messages up to
MPIX_STAGE_CHUNK claim a slot of the rank's device arena inside the kernel;
larger ones use a host-provided staging buffer. Both must deliver the exact
bytes, in order, and recycle their buffers.
"""
import pytest
import torch

from paper_2208_13707_b200 import mpix
from tests.gpu_util import gpu_world, sync_all

pytestmark = pytest.mark.gpu


def rand_bytes(n, seed, device=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.randint(0, 256, (max(n, 1),), dtype=torch.uint8, generator=g)[:n].to(device)


@pytest.mark.parametrize("n", [4097, 65536, (1 << 20) + 5, (6 << 20) + 1])
def test_staged_self_sends_then_recvs(n, monkeypatch):
    """K blocking self-sends before any receive (all staged), then K receives
    in order; 6 MiB exceeds the 4 MiB arena chunk (host staging path)."""
    K = 5
    with gpu_world(1) as (w, ctx):
        c = ctx[0].comm
        src = [rand_bytes(n, 100 + i) for i in range(K)]
        dst = [torch.zeros(n, dtype=torch.uint8, device=0) for _ in range(K)]
        torch.cuda.synchronize()
        for rep in range(3):  # arena slots are released and reused
            for i in range(K):
                c.send_enqueue(src[i], n, mpix.MPI_BYTE, 0, 6)
            for i in range(K):
                c.recv_enqueue(dst[i], n, mpix.MPI_BYTE, 0, 6)
            sync_all(ctx)
            for i in range(K):
                assert torch.equal(dst[i].cpu(), src[i].cpu()), (rep, i)
                dst[i].zero_()
            assert mpix.rank_error(0) == 0


def test_arena_smaller_than_outstanding_sends_uses_recycled_slots(monkeypatch):
    """With 2 arena slots, a ping-pong of staged sends recycles the two
    slots across many iterations (each receive releases its slot)."""
    monkeypatch.setenv("MPIX_STAGE_SLOTS", "2")
    n, iters = 100_000, 50
    with gpu_world(2) as (w, ctx):
        buf = [rand_bytes(n, 7 + r) for r in range(2)]
        first = buf[0].clone()
        torch.cuda.synchronize()

        def body(r):
            c = ctx[r].comm
            for _ in range(iters):
                if r == 0:
                    c.send_enqueue(buf[0], n, mpix.MPI_BYTE, 1, 1)
                    c.recv_enqueue(buf[0], n, mpix.MPI_BYTE, 1, 2)
                else:
                    c.recv_enqueue(buf[1], n, mpix.MPI_BYTE, 0, 1)
                    c.send_enqueue(buf[1], n, mpix.MPI_BYTE, 0, 2)

        w.run_ranks(body)
        sync_all(ctx)
        assert torch.equal(buf[0].cpu(), first.cpu())
        assert torch.equal(buf[1].cpu(), first.cpu())
        assert mpix.rank_error(0) == 0 and mpix.rank_error(1) == 0


def test_staged_head_to_head_blocking_sends():
    """Both ranks Send_enqueue first, then Recv_enqueue: completes only
    because sends stage (the reference's eager contract)."""
    n = 2 << 20
    with gpu_world(2) as (w, ctx):
        src = [rand_bytes(n, 200 + r) for r in range(2)]
        dst = [torch.zeros(n, dtype=torch.uint8, device=0) for _ in range(2)]
        torch.cuda.synchronize()

        def body(r):
            c = ctx[r].comm
            c.send_enqueue(src[r], n, mpix.MPI_BYTE, 1 - r, 3)
            c.recv_enqueue(dst[r], n, mpix.MPI_BYTE, 1 - r, 3)

        for _ in range(4):
            w.run_ranks(body)
        sync_all(ctx)
        for r in range(2):
            assert torch.equal(dst[r].cpu(), src[1 - r].cpu())
