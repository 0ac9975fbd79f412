"""GPU parity tests of the enqueue point-to-point path.

Every test calls the C ABI through the ctypes binding; payload bytes must be
bit-identical to what was sent (the reference delivers with memcpy,
proj/src/endpoint.cpp:17-18), truncation follows endpoint.cpp:17-24.
"""
import numpy as np
import pytest
import torch

from paper_2208_13707_b200 import mpix
from tests.gpu_util import gpu_world, sync_all

pytestmark = pytest.mark.gpu

SIZES = [0, 1, 8, 15, 4096, 4097, 65536 + 3, 1 << 20, (8 << 20) + 16]


def rand_bytes(n, seed, device=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.randint(0, 256, (max(n, 1),), dtype=torch.uint8, generator=g)[:n].to(device)


@pytest.mark.parametrize("n", SIZES)
def test_loopback_isend_irecv_waitall(n):
    """1 GPU loopback: Isend/Irecv/Waitall on one stream (SURVEY §8d cfg2, 1 GPU)."""
    with gpu_world(1) as (w, ctx):
        c = ctx[0]
        src = rand_bytes(n, 1)
        dst = torch.zeros(max(n, 1), dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        r1 = c.comm.isend_enqueue(src, n, mpix.MPI_BYTE, 0, 7)
        r2 = c.comm.irecv_enqueue(dst, n, mpix.MPI_BYTE, 0, 7)
        mpix.waitall_enqueue([r1, r2])
        sync_all(ctx)
        assert torch.equal(dst[:n].cpu(), src.cpu())


@pytest.mark.parametrize("n", SIZES)
def test_self_send_then_recv_same_stream(n):
    """Appendix A1: a blocking self-send then self-recv on the same stream
    completes with identical bytes (eager/staged sends, proc_p2p.cpp:42-62)."""
    with gpu_world(1) as (w, ctx):
        c = ctx[0]
        src = rand_bytes(n, 2)
        dst = torch.zeros(max(n, 1), dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        c.comm.send_enqueue(src, n, mpix.MPI_BYTE, 0, 3)
        c.comm.recv_enqueue(dst, n, mpix.MPI_BYTE, 0, 3)
        sync_all(ctx)
        assert torch.equal(dst[:n].cpu(), src.cpu())


def test_irecv_before_isend_same_stream():
    with gpu_world(1) as (w, ctx):
        c = ctx[0]
        n = 3 << 20
        src = rand_bytes(n, 3)
        dst = torch.zeros(n, dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        r2 = c.comm.irecv_enqueue(dst, n, mpix.MPI_BYTE, 0, 1)
        r1 = c.comm.isend_enqueue(src, n, mpix.MPI_BYTE, 0, 1)
        mpix.waitall_enqueue([r1, r2])
        sync_all(ctx)
        assert torch.equal(dst.cpu(), src.cpu())


@pytest.mark.parametrize("n", [8, 4096, 1 << 20, 5 << 20])
def test_two_rank_pingpong(n):
    """cfg1 shape: 2 ranks (streams) ping-pong Send/Recv_enqueue; rank 0 sends
    x, rank 1 receives and sends it back; repeated with fresh data."""
    with gpu_world(2) as (w, ctx):
        a, b = ctx
        x = rand_bytes(n, 4)
        back = torch.zeros(max(n, 1), dtype=torch.uint8, device=0)
        mid = torch.zeros(max(n, 1), dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        iters = 5

        def rank(r):
            for it in range(iters):
                if r == 0:
                    a.comm.send_enqueue(x, n, mpix.MPI_BYTE, 1, 10)
                    a.comm.recv_enqueue(back, n, mpix.MPI_BYTE, 1, 11)
                else:
                    b.comm.recv_enqueue(mid, n, mpix.MPI_BYTE, 0, 10)
                    b.comm.send_enqueue(mid, n, mpix.MPI_BYTE, 0, 11)

        w.run_ranks(rank)
        sync_all(ctx)
        assert torch.equal(back[:n].cpu(), x.cpu())
        assert torch.equal(mid[:n].cpu(), x.cpu())


def test_head_to_head_blocking_sends_complete():
    """Both ranks Send_enqueue then Recv_enqueue (completes because
    sends are eager); large size exercises the staged path."""
    for n in (64, 2 << 20):
        with gpu_world(2) as (w, ctx):
            bufs = [rand_bytes(n, 10 + r) for r in range(2)]
            outs = [torch.zeros(n, dtype=torch.uint8, device=0) for _ in range(2)]
            torch.cuda.synchronize()

            def rank(r):
                c = ctx[r].comm
                c.send_enqueue(bufs[r], n, mpix.MPI_BYTE, 1 - r, 0)
                c.recv_enqueue(outs[r], n, mpix.MPI_BYTE, 1 - r, 0)

            w.run_ranks(rank)
            sync_all(ctx)
            assert torch.equal(outs[0].cpu(), bufs[1].cpu())
            assert torch.equal(outs[1].cpu(), bufs[0].cpu())


@pytest.mark.parametrize("n,cap", [(100, 40), (10000, 4096), (3 << 20, 1 << 20), (16, 0)])
def test_truncation(n, cap):
    """Appendix A2: capacity < message -> first `cap` bytes delivered, the
    rest of the receive buffer untouched, the stream continues."""
    with gpu_world(1) as (w, ctx):
        c = ctx[0]
        src = rand_bytes(n, 5)
        dst = torch.full((cap + 64,), 0xAB, dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        r1 = c.comm.isend_enqueue(src, n, mpix.MPI_BYTE, 0, 2)
        r2 = c.comm.irecv_enqueue(dst, cap, mpix.MPI_BYTE, 0, 2)
        mpix.waitall_enqueue([r1, r2])
        sync_all(ctx)
        got = dst.cpu()
        assert torch.equal(got[:cap], src.cpu()[:cap])
        assert bool((got[cap:] == 0xAB).all())


def test_zero_count_leaves_buffer_untouched():
    """Appendix A3: count=0 completes; the receive buffer is untouched."""
    with gpu_world(2) as (w, ctx):
        dst = torch.full((32,), 0x5A, dtype=torch.uint8, device=0)
        src = torch.zeros(32, dtype=torch.uint8, device=0)
        torch.cuda.synchronize()

        def rank(r):
            if r == 0:
                ctx[0].comm.send_enqueue(src, 0, mpix.MPI_BYTE, 1, 4)
            else:
                ctx[1].comm.recv_enqueue(dst, 0, mpix.MPI_BYTE, 0, 4)

        w.run_ranks(rank)
        sync_all(ctx)
        assert bool((dst.cpu() == 0x5A).all())


def test_non_overtaking_same_tag_and_interleaved_tags():
    """Appendix A10: three isends with the same tag are received in order even
    when receives for another tag are posted in between; tags may be received
    in a different order than sent (per-tag matching)."""
    with gpu_world(2) as (w, ctx):
        vals = [10, 20, 30]
        srcs = [torch.full((256,), v, dtype=torch.int32, device=0) for v in vals]
        five = torch.full((256,), 5, dtype=torch.int32, device=0)
        outs = [torch.zeros(256, dtype=torch.int32, device=0) for _ in range(3)]
        out5 = torch.zeros(256, dtype=torch.int32, device=0)
        torch.cuda.synchronize()

        def rank(r):
            c = ctx[r].comm
            if r == 0:
                reqs = [c.isend_enqueue(s, 256, mpix.MPI_INT, 1, 1) for s in srcs]
                reqs.append(c.isend_enqueue(five, 256, mpix.MPI_INT, 1, 5))
                mpix.waitall_enqueue(reqs)
            else:
                reqs = [c.irecv_enqueue(out5, 256, mpix.MPI_INT, 0, 5)]
                reqs += [c.irecv_enqueue(o, 256, mpix.MPI_INT, 0, 1) for o in outs]
                mpix.waitall_enqueue(reqs)

        w.run_ranks(rank)
        sync_all(ctx)
        assert [int(o[0]) for o in outs] == vals
        assert int(out5[0]) == 5 and bool((out5 == 5).all())


def test_window_of_isends_exceeding_ring():
    """More outstanding messages per pair than ring slots: posting waits for
    slots to drain, which the peer's receives do (no deadlock)."""
    with gpu_world(2) as (w, ctx):
        R = mpix.config()["ring_slots"]
        m = R + 37
        src = torch.arange(m * 4, dtype=torch.int32, device=0).reshape(m, 4)
        dst = torch.zeros_like(src)
        torch.cuda.synchronize()

        def rank(r):
            c = ctx[r].comm
            if r == 0:
                reqs = [c.isend_enqueue(src[i], 4, mpix.MPI_INT, 1, i % 3) for i in range(m)]
            else:
                reqs = [c.irecv_enqueue(dst[i], 4, mpix.MPI_INT, 0, i % 3) for i in range(m)]
            mpix.waitall_enqueue(reqs)

        w.run_ranks(rank)
        sync_all(ctx)
        assert torch.equal(dst.cpu(), src.cpu())


def test_listing2_saxpy():
    """SPEC.md:420 / PAPER.md Listing 2: rank 0 sends x (all 1.0); rank 1
    receives into x then SAXPY with a=2, y=2 -> every element 4.0 (N=1024)."""
    N = 1024
    with gpu_world(2) as (w, ctx):
        x0 = torch.ones(N, dtype=torch.float32, device=0)
        x1 = torch.zeros(N, dtype=torch.float32, device=0)
        y1 = torch.full((N,), 2.0, dtype=torch.float32, device=0)
        torch.cuda.synchronize()

        def rank(r):
            c = ctx[r]
            if r == 0:
                c.comm.send_enqueue(x0, N, mpix.MPI_FLOAT, 1, 0)
            else:
                c.comm.recv_enqueue(x1, N, mpix.MPI_FLOAT, 0, 0)
                mpix.testing.saxpy(N, 2.0, x1, y1, c.stream)

        w.run_ranks(rank)
        sync_all(ctx)
        assert bool((y1.cpu() == 4.0).all())


def test_enqueue_returns_while_peer_is_delayed():
    """SPEC.md:436 / Appendix A8: enqueue calls never block on the peer. Rank
    1's stream is held by a 200 ms device delay; rank 0's calls return at
    once and its stream completes only after the peer's receive ran."""
    import time
    with gpu_world(2) as (w, ctx):
        n = 1 << 20
        src = rand_bytes(n, 6)
        dst = torch.zeros(n, dtype=torch.uint8, device=0)
        back = torch.zeros(n, dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        mpix.testing.delay(200_000_000, ctx[1].stream)
        t0 = time.perf_counter()
        ctx[0].comm.send_enqueue(src, n, mpix.MPI_BYTE, 1, 0)
        ctx[0].comm.recv_enqueue(back, n, mpix.MPI_BYTE, 1, 1)
        r = ctx[0].comm.isend_enqueue(src, n, mpix.MPI_BYTE, 1, 2)
        mpix.wait_enqueue(r)
        t_call = time.perf_counter() - t0
        ctx[1].comm.recv_enqueue(dst, n, mpix.MPI_BYTE, 0, 0)
        ctx[1].comm.send_enqueue(dst, n, mpix.MPI_BYTE, 0, 1)
        ctx[1].comm.recv_enqueue(dst, n, mpix.MPI_BYTE, 0, 2)
        sync_all(ctx)
        t_all = time.perf_counter() - t0
        assert t_call < 0.05, t_call
        assert t_all > 0.15, t_all
        assert torch.equal(back.cpu(), src.cpu())


def test_fifo_order_in_stream():
    """SPEC.md:434 (queue FIFO): a kernel enqueued after Recv_enqueue sees the
    received data; one enqueued before sees the old data."""
    with gpu_world(2) as (w, ctx):
        N = 4096
        x = torch.full((N,), 3.0, device=0)
        y = torch.zeros(N, device=0)
        before = torch.zeros(N, device=0)
        after = torch.zeros(N, device=0)
        torch.cuda.synchronize()
        s1 = ctx[1].stream
        with torch.cuda.stream(s1):
            before.copy_(y)
        ctx[1].comm.recv_enqueue(y, N, mpix.MPI_FLOAT, 0, 9)
        with torch.cuda.stream(s1):
            after.copy_(y)
        ctx[0].comm.send_enqueue(x, N, mpix.MPI_FLOAT, 1, 9)
        sync_all(ctx)
        assert bool((before.cpu() == 0).all())
        assert bool((after.cpu() == 3.0).all())


def test_many_pairs_four_ranks():
    """All-to-all of distinct payloads among 4 ranks, mixed blocking/non-blocking."""
    P = 4
    with gpu_world(P) as (w, ctx):
        n = 70000
        src = [[rand_bytes(n, 100 + 10 * s + d) for d in range(P)] for s in range(P)]
        dst = [[torch.zeros(n, dtype=torch.uint8, device=0) for _ in range(P)] for _ in range(P)]
        torch.cuda.synchronize()

        def rank(r):
            c = ctx[r].comm
            reqs = []
            for d in range(P):
                reqs.append(c.irecv_enqueue(dst[r][d], n, mpix.MPI_BYTE, d, 3))
            for d in range(P):
                reqs.append(c.isend_enqueue(src[r][d], n, mpix.MPI_BYTE, d, 3))
            mpix.waitall_enqueue(reqs)

        w.run_ranks(rank)
        sync_all(ctx)
        for r in range(P):
            for s in range(P):
                assert torch.equal(dst[r][s].cpu(), src[s][r].cpu()), (r, s)
