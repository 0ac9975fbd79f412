"""GPU tests of CUDA-Graph capture of enqueued operations.

The paper treats the enqueue APIs as work placed in a GPU execution queue,
and names the execution graph as that queue's generalisation
(PAPER.md:228-237). Here, each rank captures its stream into a CUDA graph and replays it K
times. Inside the graph:
- a producer kernel fills the send buffer from a device iteration word;
- the enqueued communication follows;
- a consumer kernel checks the received data for that iteration;
- a final kernel advances the iteration word.
So every replay moves new values and is checked on the device. A
graph-capturable comm (MPIX_GRAPH=1 or the "mpix_graph" stream hint) takes
its sequence numbers from device counters, so eager operations interleaved
with the replays stay matched.
"""
import os
import threading

import pytest
import torch

from paper_2208_13707_b200 import mpix
from tests.gpu_util import gpu_world, sync_all

pytestmark = pytest.mark.gpu

K = 12  # replays


@pytest.fixture(autouse=True)
def _static_matching_only():
    # graph-capturable comms use static matching
    if os.environ.get("MPIX_MATCHING") == "dynamic":
        pytest.skip("graph capture needs static matching")


@pytest.fixture
def graph_env(monkeypatch):
    monkeypatch.setenv("MPIX_GRAPH", "1")


class Replay:
    """Per-rank iteration word + mismatch counter, and the captured graph."""

    def __init__(self, ctx):
        self.ctx = ctx
        self.it = torch.zeros(1, dtype=torch.int32, device=ctx.device)
        self.bad = torch.zeros(1, dtype=torch.int64, device=ctx.device)
        self.exec = None

    def capture(self, body):
        s = self.ctx.stream
        s.synchronize()
        mpix.testing.graph_begin(s)
        try:
            body()
        finally:
            self.exec = mpix.testing.graph_end(s)

    def launch(self, k):
        for _ in range(k):
            mpix.testing.graph_launch(self.exec, self.ctx.stream)

    def close(self):
        if self.exec:
            mpix.testing.graph_destroy(self.exec)
            self.exec = None


def eager_ring(w, ctx, n, tag):
    """One eager (uncaptured) ring exchange, host-checked."""
    P = len(ctx)
    outs = [None] * P

    def body(r):
        c = ctx[r]
        src = torch.full((n,), float(1000 * tag + r), device=c.device)
        dst = torch.zeros(n, device=c.device)
        c.stream.synchronize()
        with torch.cuda.stream(c.stream):
            rq = [c.comm.isend_enqueue(src, n, mpix.MPI_FLOAT, (r + 1) % P, tag),
                  c.comm.irecv_enqueue(dst, n, mpix.MPI_FLOAT, (r - 1) % P, tag)]
            mpix.waitall_enqueue(rq)
        c.stream.synchronize()
        outs[r] = (src, dst)

    w.run_ranks(body)
    for r in range(P):
        assert torch.all(outs[r][1] == float(1000 * tag + (r - 1) % P)).item(), r


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("n", [2, 1024, 262144], ids=["8B", "4KiB", "1MiB"])
def test_captured_ring_exchange_replays(P, n, graph_env):
    """Isend/Irecv/Waitall ring captured per rank; K replays, each checked
    on the device; eager exchanges before and after on the same comm."""
    with gpu_world(P) as (w, ctx):
        eager_ring(w, ctx, 64, tag=1)
        reps = [Replay(c) for c in ctx]
        bufs = [(torch.zeros(n, device=c.device), torch.zeros(n, device=c.device)) for c in ctx]

        def cap(r):
            c, rp = ctx[r], reps[r]
            src, dst = bufs[r]
            left = (r - 1) % P

            def body():
                mpix.testing.iter_fill(src, n, rp.it, float(r + 1), 1.0, c.stream)
                rq = [c.comm.irecv_enqueue(dst, n, mpix.MPI_FLOAT, left, 7),
                      c.comm.isend_enqueue(src, n, mpix.MPI_FLOAT, (r + 1) % P, 7)]
                mpix.waitall_enqueue(rq)
                mpix.testing.iter_check(dst, n, rp.it, float(left + 1), 1.0, rp.bad, c.stream)
                mpix.testing.iter_bump(rp.it, c.stream)

            rp.capture(body)

        w.run_ranks(cap)
        w.run_ranks(lambda r: reps[r].launch(K))
        sync_all(ctx)
        for rp in reps:
            assert rp.it.item() == K
            assert rp.bad.item() == 0
        eager_ring(w, ctx, 64, tag=2)  # counters still agree after the replays
        w.run_ranks(lambda r: reps[r].launch(2))
        sync_all(ctx)
        assert all(rp.it.item() == K + 2 and rp.bad.item() == 0 for rp in reps)
        for rp in reps:
            rp.close()


@pytest.mark.parametrize("n", [16, 524288], ids=["64B-eager", "2MiB-staged"])
def test_captured_blocking_pingpong(n, graph_env):
    """Send_enqueue / Recv_enqueue (blocking) captured on both sides of a
    ping-pong: eager sends, and large sends through the device staging arena."""
    with gpu_world(2) as (w, ctx):
        reps = [Replay(c) for c in ctx]
        bufs = [(torch.zeros(n, device=0), torch.zeros(n, device=0)) for _ in ctx]

        def cap(r):
            c, rp = ctx[r], reps[r]
            src, dst = bufs[r]
            peer = 1 - r

            def body():
                mpix.testing.iter_fill(src, n, rp.it, float(r + 1), 2.0, c.stream)
                if r == 0:
                    c.comm.send_enqueue(src, n, mpix.MPI_FLOAT, peer, 3)
                    c.comm.recv_enqueue(dst, n, mpix.MPI_FLOAT, peer, 4)
                else:
                    c.comm.recv_enqueue(dst, n, mpix.MPI_FLOAT, peer, 3)
                    c.comm.send_enqueue(src, n, mpix.MPI_FLOAT, peer, 4)
                mpix.testing.iter_check(dst, n, rp.it, float(peer + 1), 2.0, rp.bad, c.stream)
                mpix.testing.iter_bump(rp.it, c.stream)

            rp.capture(body)

        w.run_ranks(cap)
        w.run_ranks(lambda r: reps[r].launch(K))
        sync_all(ctx)
        assert [rp.it.item() for rp in reps] == [K, K]
        assert [rp.bad.item() for rp in reps] == [0, 0]
        for rp in reps:
            rp.close()


@pytest.mark.parametrize("n", [1024, 65536], ids=["4KiB", "256KiB"])
def test_captured_self_messages(n, graph_env):
    """One rank, self-messages (no host pairing on a graph-capturable comm):
    a window of 4 Isend/Irecv pairs + Waitall per replay."""
    with gpu_world(1) as (w, ctx):
        c = ctx[0]
        rp = Replay(c)
        src = [torch.zeros(n, device=0) for _ in range(4)]
        dst = [torch.zeros(n, device=0) for _ in range(4)]

        def body():
            rq = []
            for j in range(4):
                mpix.testing.iter_fill(src[j], n, rp.it, float(j + 1), 1.0, c.stream)
            for j in range(4):
                rq.append(c.comm.isend_enqueue(src[j], n, mpix.MPI_FLOAT, 0, 5))
                rq.append(c.comm.irecv_enqueue(dst[j], n, mpix.MPI_FLOAT, 0, 5))
            mpix.waitall_enqueue(rq)
            for j in range(4):  # same tag: message order is preserved (non-overtaking)
                mpix.testing.iter_check(dst[j], n, rp.it, float(j + 1), 1.0, rp.bad, c.stream)
            mpix.testing.iter_bump(rp.it, c.stream)

        w.run_ranks(lambda r: rp.capture(body))
        w.run_ranks(lambda r: rp.launch(K))
        sync_all(ctx)
        assert rp.it.item() == K and rp.bad.item() == 0
        rp.close()


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("n", [1024, 1 << 20], ids=["4KiB-fused", "4MiB-twoshot"])
def test_captured_allreduce(P, n, graph_env):
    """Allreduce_enqueue captured between producer and consumer kernels:
    x_r = (it+1)(r+1) + i%7, so the sum is (it+1)P(P+1)/2 + P(i%7), exact."""
    with gpu_world(P) as (w, ctx):
        reps = [Replay(c) for c in ctx]
        bufs = [(torch.zeros(n, device=0), torch.zeros(n, device=0)) for _ in ctx]
        tri = P * (P + 1) / 2

        def cap(r):
            c, rp = ctx[r], reps[r]
            x, y = bufs[r]

            def body():
                mpix.testing.iter_fill(x, n, rp.it, float(r + 1), 1.0, c.stream)
                c.comm.allreduce_enqueue(x, y, n, mpix.MPI_FLOAT)
                mpix.testing.iter_check(y, n, rp.it, tri, float(P), rp.bad, c.stream)
                mpix.testing.iter_bump(rp.it, c.stream)

            rp.capture(body)

        w.run_ranks(cap)
        w.run_ranks(lambda r: reps[r].launch(K))
        sync_all(ctx)
        assert all(rp.it.item() == K for rp in reps)
        assert [rp.bad.item() for rp in reps] == [0] * P
        # an eager allreduce on the same comm afterwards (epoch counter agrees)
        outs = [torch.zeros(64, device=0) for _ in ctx]

        def eager(r):
            with torch.cuda.stream(ctx[r].stream):
                ctx[r].comm.allreduce_enqueue(torch.full((64,), float(r), device=0), outs[r], 64,
                                              mpix.MPI_FLOAT)
            ctx[r].stream.synchronize()

        w.run_ranks(eager)
        assert all(torch.all(o == P * (P - 1) / 2).item() for o in outs)
        for rp in reps:
            rp.close()


def test_captured_bcast_and_allgather(graph_env):
    P, n = 3, 4096
    with gpu_world(P) as (w, ctx):
        reps = [Replay(c) for c in ctx]
        bb = [torch.zeros(n, device=0) for _ in ctx]
        src = [torch.zeros(n, device=0) for _ in ctx]
        ag = [torch.zeros(P * n, device=0) for _ in ctx]

        def cap(r):
            c, rp = ctx[r], reps[r]

            def body():
                if r == 1:
                    mpix.testing.iter_fill(bb[r], n, rp.it, 5.0, 1.0, c.stream)
                c.comm.bcast_enqueue(bb[r], n, mpix.MPI_FLOAT, root=1)
                mpix.testing.iter_check(bb[r], n, rp.it, 5.0, 1.0, rp.bad, c.stream)
                mpix.testing.iter_fill(src[r], n, rp.it, float(r + 1), 0.0, c.stream)
                c.comm.allgather_enqueue(src[r], ag[r], n, mpix.MPI_FLOAT)
                for q in range(P):
                    mpix.testing.iter_check(ag[r][q * n:(q + 1) * n], n, rp.it, float(q + 1), 0.0,
                                            rp.bad, c.stream)
                mpix.testing.iter_bump(rp.it, c.stream)

            rp.capture(body)

        w.run_ranks(cap)
        w.run_ranks(lambda r: reps[r].launch(K))
        sync_all(ctx)
        assert [rp.bad.item() for rp in reps] == [0] * P
        assert all(rp.it.item() == K for rp in reps)
        for rp in reps:
            rp.close()


def test_captured_alltoall(graph_env):
    P, n = 3, 2048
    with gpu_world(P) as (w, ctx):
        reps = [Replay(c) for c in ctx]
        sb = [torch.zeros(P * n, device=0) for _ in ctx]
        rb = [torch.zeros(P * n, device=0) for _ in ctx]

        def cap(r):
            c, rp = ctx[r], reps[r]

            def body():
                for q in range(P):  # block q, for rank q: (it+1)(10r+q+1) + i%7
                    mpix.testing.iter_fill(sb[r][q * n:(q + 1) * n], n, rp.it,
                                           float(10 * r + q + 1), 1.0, c.stream)
                c.comm.alltoall_enqueue(sb[r], rb[r], n, mpix.MPI_FLOAT)
                for q in range(P):  # block q of mine came from rank q
                    mpix.testing.iter_check(rb[r][q * n:(q + 1) * n], n, rp.it,
                                            float(10 * q + r + 1), 1.0, rp.bad, c.stream)
                mpix.testing.iter_bump(rp.it, c.stream)

            rp.capture(body)

        w.run_ranks(cap)
        w.run_ranks(lambda r: reps[r].launch(K))
        sync_all(ctx)
        assert [rp.bad.item() for rp in reps] == [0] * P
        assert all(rp.it.item() == K for rp in reps)
        for rp in reps:
            rp.close()


def test_graph_hint_and_capture_rules():
    """The "mpix_graph" stream hint makes one comm graph-capturable; on a
    comm without it, capture is refused (UNSUPPORTED) rather than replaying
    stale sequence numbers; captured requests are waited in their graph."""
    w = mpix.World(1, [0])
    try:
        out = {}

        def body(r):
            s = mpix.testing.new_stream(0)
            plain = w.comm(0).stream_comm_create(mpix.Stream.from_cuda(s, mpix_graph="0"))
            s2 = mpix.testing.new_stream(0)
            gcomm = w.comm(0).stream_comm_create(mpix.Stream.from_cuda(s2, mpix_graph="1"))
            x = torch.ones(16, device=0)
            y = torch.zeros(16, device=0)
            codes = []
            # plain comm: a blocking op and a collective refuse to be captured
            mpix.testing.graph_begin(s)
            for fn in (lambda: plain.send_enqueue(x, 16, mpix.MPI_FLOAT, 0, 1),
                       lambda: plain.allreduce_enqueue(x, y, 16, mpix.MPI_FLOAT)):
                try:
                    fn()
                    codes.append("ok")
                except mpix.MPIXError as e:
                    codes.append(e.name)
            ex = mpix.testing.graph_end(s)
            mpix.testing.graph_destroy(ex)
            # graph comm: capture works; its requests cannot be waited outside
            it = torch.zeros(1, dtype=torch.int32, device=0)
            mpix.testing.graph_begin(s2)
            try:
                rq = [gcomm.isend_enqueue(x, 16, mpix.MPI_FLOAT, 0, 2),
                      gcomm.irecv_enqueue(y, 16, mpix.MPI_FLOAT, 0, 2)]
                mpix.waitall_enqueue(rq)
                mpix.testing.iter_bump(it, s2)
            finally:
                ex = mpix.testing.graph_end(s2)
            for _ in range(3):
                mpix.testing.graph_launch(ex, s2)
            s2.synchronize()
            mpix.testing.graph_destroy(ex)
            out["codes"] = codes
            out["y"] = y.clone()
            out["it"] = it.item()
            plain.free()
            gcomm.free()

        w.run_ranks(body)
        assert out["codes"] == ["UNSUPPORTED", "UNSUPPORTED"]
        assert out["it"] == 3
        assert torch.all(out["y"] == 1).item()
    finally:
        torch.cuda.synchronize()
        w.finalize()


def test_replays_interleaved_with_eager_traffic(graph_env):
    """Replays and eager operations alternate on the same comm and tag: the
    device counters make both sides agree on every message's sequence."""
    P, n = 2, 4096
    with gpu_world(P) as (w, ctx):
        reps = [Replay(c) for c in ctx]
        bufs = [(torch.zeros(n, device=0), torch.zeros(n, device=0)) for _ in ctx]

        def cap(r):
            c, rp = ctx[r], reps[r]
            src, dst = bufs[r]

            def body():
                mpix.testing.iter_fill(src, n, rp.it, float(r + 1), 1.0, c.stream)
                rq = [c.comm.isend_enqueue(src, n, mpix.MPI_FLOAT, 1 - r, 9),
                      c.comm.irecv_enqueue(dst, n, mpix.MPI_FLOAT, 1 - r, 9)]
                mpix.waitall_enqueue(rq)
                mpix.testing.iter_check(dst, n, rp.it, float(2 - r), 1.0, rp.bad, c.stream)
                mpix.testing.iter_bump(rp.it, c.stream)

            rp.capture(body)

        w.run_ranks(cap)
        lock = threading.Lock()
        got = []

        def mixed(r):
            c = ctx[r]
            for k in range(4):
                reps[r].launch(1)
                e_src = torch.full((32,), float(100 * k + r), device=0)
                e_dst = torch.zeros(32, device=0)
                with torch.cuda.stream(c.stream):  # same tag as the graph's messages
                    rq = [c.comm.isend_enqueue(e_src, 32, mpix.MPI_FLOAT, 1 - r, 9),
                          c.comm.irecv_enqueue(e_dst, 32, mpix.MPI_FLOAT, 1 - r, 9)]
                    mpix.waitall_enqueue(rq)
                c.stream.synchronize()
                with lock:
                    got.append((r, k, e_dst[0].item()))

        w.run_ranks(mixed)
        sync_all(ctx)
        assert all(rp.it.item() == 4 and rp.bad.item() == 0 for rp in reps)
        for r, k, v in got:
            assert v == 100 * k + (1 - r), (r, k, v)
        for rp in reps:
            rp.close()
