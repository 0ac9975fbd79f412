"""GPU tests of coalesced launches (host-side op batching).

Inline-sized non-blocking operations are held per CUDA stream and launched
together by the next ordering call. Results must not depend on it: every
test checks payload bytes against what was sent, and the same program is
run with batching disabled (MPIX_BATCH=0) where the two could differ.
"""
import pytest
import torch

from paper_2208_13707_b200 import mpix
from tests.gpu_util import gpu_world, sync_all

pytestmark = pytest.mark.gpu


def rand_bytes(n, seed, device=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.randint(0, 256, (max(n, 1),), dtype=torch.uint8, generator=g)[:n].to(device)


@pytest.fixture(params=["1", "0"], ids=["batch", "nobatch"])
def batch_env(request, monkeypatch):
    monkeypatch.setenv("MPIX_BATCH", request.param)
    # launch counts below assume no held batch ages past the flusher's
    # deadline while the Python loop enqueues (a progress guarantee that
    # these tests never need)
    monkeypatch.setenv("MPIX_FLUSH_US", "2000000")
    return request.param == "1"


def test_window_of_one_launch(batch_env):
    """W Isend + W Irecv + Waitall on one stream: a single launch when the
    window fits one batch (2W <= 64 ops, 2W <= 128 waits)."""
    W, n = 32, 64
    with gpu_world(1) as (w, ctx):
        c = ctx[0].comm
        src = [rand_bytes(n, 10 + i) for i in range(W)]
        dst = torch.zeros((W, n), dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        l0 = mpix.launch_count()
        reqs = []
        for i in range(W):
            reqs.append(c.isend_enqueue(src[i], n, mpix.MPI_BYTE, 0, i))
            reqs.append(c.irecv_enqueue(dst[i], n, mpix.MPI_BYTE, 0, i))
        mpix.waitall_enqueue(reqs)
        launches = mpix.launch_count() - l0
        sync_all(ctx)
        for i in range(W):
            assert torch.equal(dst[i].cpu(), src[i].cpu()), i
        assert launches == (1 if batch_env else 2 * W + 1)


@pytest.mark.parametrize("W", [65, 120])
def test_window_larger_than_a_batch(W, batch_env):
    """More operations than one batch holds (intermediate flushes) and more
    requests than one wait launch carries (chunked waits). W stays within the
    ring (R = 128 unmatched posts per comm, pair and direction): a stream
    that posts more self-receives than that before their sends waits for a
    slot that only a later operation of the same stream can free."""
    n = 24
    with gpu_world(1) as (w, ctx):
        c = ctx[0].comm
        src = rand_bytes(W * n, 5).view(W, n)
        dst = torch.zeros((W, n), dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        reqs = []
        for i in range(W):
            reqs.append(c.irecv_enqueue(dst[i], n, mpix.MPI_BYTE, 0, 1))  # same tag: order
        for i in range(W):
            reqs.append(c.isend_enqueue(src[i], n, mpix.MPI_BYTE, 0, 1))
        mpix.waitall_enqueue(reqs)
        sync_all(ctx)
        assert torch.equal(dst.cpu(), src.cpu())


def test_head_to_head_isend_then_blocking_recv(batch_env):
    """A: Isend(B) Recv(B); B: Isend(A) Recv(A). The held Isend joins the
    blocking Recv's launch, so neither side waits on a send that was never
    launched."""
    n = 4096 + 7
    with gpu_world(2) as (w, ctx):
        src = [rand_bytes(n, 20 + r) for r in range(2)]
        dst = [torch.zeros(n, dtype=torch.uint8, device=0) for _ in range(2)]
        torch.cuda.synchronize()
        reqs = [None, None]

        def body(r):
            c = ctx[r].comm
            reqs[r] = c.isend_enqueue(src[r], n, mpix.MPI_BYTE, 1 - r, 4)
            c.recv_enqueue(dst[r], n, mpix.MPI_BYTE, 1 - r, 4)
            mpix.wait_enqueue(reqs[r])

        for _ in range(3):
            w.run_ranks(body)
        sync_all(ctx)
        for r in range(2):
            assert torch.equal(dst[r].cpu(), src[1 - r].cpu())


def test_small_ops_then_large_op_keep_stream_order(batch_env):
    """Held small Irecvs are launched before a large Isend/Irecv that follows
    them on the same stream; tag order (non-overtaking) is preserved."""
    small, big = 100, (4 << 20) + 3
    with gpu_world(1) as (w, ctx):
        c = ctx[0].comm
        s_src = [rand_bytes(small, 30 + i) for i in range(3)]
        b_src = rand_bytes(big, 40)
        s_dst = [torch.zeros(small, dtype=torch.uint8, device=0) for _ in range(3)]
        b_dst = torch.zeros(big, dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        reqs = [c.irecv_enqueue(s_dst[i], small, mpix.MPI_BYTE, 0, 9) for i in range(3)]
        reqs.append(c.irecv_enqueue(b_dst, big, mpix.MPI_BYTE, 0, 9))
        reqs += [c.isend_enqueue(s_src[i], small, mpix.MPI_BYTE, 0, 9) for i in range(3)]
        reqs.append(c.isend_enqueue(b_src, big, mpix.MPI_BYTE, 0, 9))
        mpix.waitall_enqueue(reqs)
        sync_all(ctx)
        for i in range(3):
            assert torch.equal(s_dst[i].cpu(), s_src[i].cpu())
        assert torch.equal(b_dst.cpu(), b_src.cpu())


def test_allreduce_after_held_ops(batch_env):
    """An Allreduce_enqueue orders the stream: held p2p ops launch first."""
    P, n, cnt = 2, 256, 1024
    with gpu_world(P) as (w, ctx):
        src = [rand_bytes(n, 50 + r) for r in range(P)]
        dst = [torch.zeros(n, dtype=torch.uint8, device=0) for _ in range(P)]
        x = [torch.full((cnt,), float(r + 1), device=0) for r in range(P)]
        y = [torch.zeros(cnt, device=0) for _ in range(P)]
        torch.cuda.synchronize()
        reqs = {}

        def body(r):
            c = ctx[r].comm
            reqs[r] = [c.irecv_enqueue(dst[r], n, mpix.MPI_BYTE, 1 - r, 0),
                       c.isend_enqueue(src[r], n, mpix.MPI_BYTE, 1 - r, 0)]
            c.allreduce_enqueue(x[r], y[r], cnt, mpix.MPI_FLOAT)
            mpix.waitall_enqueue(reqs[r])

        w.run_ranks(body)
        sync_all(ctx)
        for r in range(P):
            assert torch.equal(dst[r].cpu(), src[1 - r].cpu())
            assert bool((y[r] == 3.0).all())


def test_comm_free_launches_held_ops():
    """MPI_Comm_free orders the stream: held operations still run."""
    n = 512
    with gpu_world(1) as (w, ctx):
        s = ctx[0].stream
        c2 = w.comm(0).stream_comm_create(mpix.Stream.from_cuda(s))
        src = rand_bytes(n, 60)
        dst = torch.zeros(n, dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        c2.isend_enqueue(src, n, mpix.MPI_BYTE, 0, 2)
        c2.irecv_enqueue(dst, n, mpix.MPI_BYTE, 0, 2)  # no wait: held until the free
        c2.free()
        s.synchronize()
        assert torch.equal(dst.cpu(), src.cpu())


def test_two_comms_one_stream_share_a_batch(batch_env):
    """Two communicators on the same CUDA stream: held operations belong to
    the stream, so a blocking call on one comm launches the other's. Rank 0
    holds an Isend on comm B, then blocks in a Recv on comm A whose matching
    Send rank 1 only issues after receiving rank 0's comm-B message."""
    n = 300
    with gpu_world(2) as (w, ctx):
        extra = {}

        def mk(r):
            extra[r] = w.comm(r).stream_comm_create(mpix.Stream.from_cuda(ctx[r].stream))

        w.run_ranks(mk)
        src_b = rand_bytes(n, 70)
        src_a = rand_bytes(n, 71)
        dst_b = torch.zeros(n, dtype=torch.uint8, device=0)
        dst_a = torch.zeros(n, dtype=torch.uint8, device=0)
        torch.cuda.synchronize()

        def body(r):
            if r == 0:
                req = extra[0].isend_enqueue(src_b, n, mpix.MPI_BYTE, 1, 1)
                ctx[0].comm.recv_enqueue(dst_a, n, mpix.MPI_BYTE, 1, 2)
                mpix.wait_enqueue(req)
            else:
                extra[1].recv_enqueue(dst_b, n, mpix.MPI_BYTE, 0, 1)
                ctx[1].comm.send_enqueue(src_a, n, mpix.MPI_BYTE, 0, 2)

        w.run_ranks(body)
        sync_all(ctx)
        assert torch.equal(dst_b.cpu(), src_b.cpu())
        assert torch.equal(dst_a.cpu(), src_a.cpu())


@pytest.mark.parametrize("sizes", [[1 << 20] * 6, [70_000, (3 << 20) + 5, 1, 4096, 65537, 8 << 20]])
def test_large_window_grouped(sizes, batch_env):
    """A halo-like window of large and small Isend/Irecv between two ranks:
    with batching it is three launches per rank (decisions, one grouped copy
    grid, completions + wait) and the bytes are exact."""
    k = len(sizes)
    with gpu_world(2) as (w, ctx):
        src = [[rand_bytes(n, 300 + 10 * r + i) for i, n in enumerate(sizes)] for r in range(2)]
        dst = [[torch.zeros(max(n, 1), dtype=torch.uint8, device=0) for n in sizes] for _ in range(2)]
        torch.cuda.synchronize()
        launches = {}

        def body(r):
            c = ctx[r].comm
            reqs = [c.irecv_enqueue(dst[r][i], n, mpix.MPI_BYTE, 1 - r, i) for i, n in enumerate(sizes)]
            reqs += [c.isend_enqueue(src[r][i], n, mpix.MPI_BYTE, 1 - r, i) for i, n in enumerate(sizes)]
            mpix.waitall_enqueue(reqs)

        l0 = mpix.launch_count()
        w.run_ranks(body)
        launches = mpix.launch_count() - l0
        sync_all(ctx)
        for r in range(2):
            for i, n in enumerate(sizes):
                assert torch.equal(dst[r][i][:n].cpu(), src[1 - r][i].cpu()), (r, i)
        if batch_env:
            assert launches == 2 * 3
        assert mpix.rank_error(0) == 0 and mpix.rank_error(1) == 0


def test_blocking_large_recv_before_send_on_same_gpu(batch_env):
    """Rank 1 blocks in a 64 MiB Recv_enqueue before rank 0 (same GPU) sends:
    the receiver's idle copy grid must not occupy the SMs the sender needs."""
    n = 64 << 20
    with gpu_world(2) as (w, ctx):
        src = rand_bytes(n, 400)
        dst = torch.zeros(n, dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        ctx[1].comm.recv_enqueue(dst, n, mpix.MPI_BYTE, 0, 8)
        mpix.testing.delay(2_000_000, ctx[0].stream)  # 2 ms: the receive is posted first
        ctx[0].comm.send_enqueue(src, n, mpix.MPI_BYTE, 1, 8)
        sync_all(ctx)
        assert torch.equal(dst.cpu(), src.cpu())
        assert mpix.rank_error(0) == 0 and mpix.rank_error(1) == 0


@pytest.mark.parametrize("n", [(1 << 20) + 3, 5 << 20])
@pytest.mark.parametrize("recv_first", [False, True])
def test_paired_self_messages(n, recv_first, batch_env):
    """Large self-messages whose send and receive meet in one batch are
    paired by the host (no descriptors): exact bytes, truncation, tag order,
    ring-slot reuse over many iterations, and blocking receives."""
    with gpu_world(1) as (w, ctx):
        c = ctx[0].comm
        src = [rand_bytes(n, 500 + i) for i in range(3)]
        dst = [torch.zeros(n, dtype=torch.uint8, device=0) for _ in range(3)]
        small = torch.zeros(n // 2, dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        for it in range(70):  # > R/2 iterations: ring slots are reused
            reqs = []
            if recv_first:
                reqs += [c.irecv_enqueue(dst[i], n, mpix.MPI_BYTE, 0, 4) for i in range(3)]
                reqs += [c.isend_enqueue(src[i], n, mpix.MPI_BYTE, 0, 4) for i in range(3)]
            else:
                reqs += [c.isend_enqueue(src[i], n, mpix.MPI_BYTE, 0, 4) for i in range(3)]
                reqs += [c.irecv_enqueue(dst[i], n, mpix.MPI_BYTE, 0, 4) for i in range(3)]
            mpix.waitall_enqueue(reqs)
        # truncation + a blocking receive closing the batch
        r = c.isend_enqueue(src[0], n, mpix.MPI_BYTE, 0, 5)
        c.recv_enqueue(small, n // 2, mpix.MPI_BYTE, 0, 5)
        mpix.wait_enqueue(r)
        sync_all(ctx)
        for i in range(3):
            assert torch.equal(dst[i].cpu(), src[i].cpu()), i
        assert torch.equal(small.cpu(), src[0][: n // 2].cpu())
        assert mpix.rank_error(0) == 0
