"""GPU: conventional (host-thread) p2p and multiplex stream p2p on GPU buffers
(proc_p2p.cpp:96-212), including
the mixed mode of Appendix A7 (a conventional send from a STREAM_NULL member
matches the peer's Recv_enqueue) and the reference's error
behaviour for these calls (proc_p2p.cpp:9-23, 96-181)."""
import pytest
import torch

from paper_2208_13707_b200 import mpix
from tests.gpu_util import gpu_world, sync_all

pytestmark = pytest.mark.gpu


def rand_bytes(n, seed, device=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.randint(0, 256, (max(n, 1),), dtype=torch.uint8, generator=g)[:n].to(device)


def err(fn):
    try:
        fn()
        return "OK"
    except mpix.MPIXError as e:
        return e.name


@pytest.mark.parametrize("n", [0, 8, 4097, (1 << 20) + 3, 6 << 20])
def test_head_to_head_blocking_send_recv_world_comm(n):
    """Both ranks MPI_Send then MPI_Recv on the world comm: completes because
    sends are eager (proc_p2p.cpp:60-62), bytes exact."""
    with gpu_world(2) as (w, ctx):
        src = [rand_bytes(n, 10 + r) for r in range(2)]
        dst = [torch.zeros(max(n, 1), dtype=torch.uint8, device=0) for _ in range(2)]
        torch.cuda.synchronize()

        def body(r):
            c = w.comm(r)
            for _ in range(3):
                c.send(src[r], n, mpix.MPI_BYTE, 1 - r, 7)
                c.recv(dst[r], n, mpix.MPI_BYTE, 1 - r, 7)

        w.run_ranks(body)
        for r in range(2):
            assert torch.equal(dst[r][:n].cpu(), src[1 - r].cpu())


def test_isend_irecv_waitall_and_request_rules():
    n = 100_000
    with gpu_world(2) as (w, ctx):
        src = [rand_bytes(n, 20 + r) for r in range(2)]
        dst = [torch.zeros(n, dtype=torch.uint8, device=0) for _ in range(2)]
        torch.cuda.synchronize()
        reqs = {}

        def body(r):
            c = w.comm(r)
            reqs[r] = [c.irecv(dst[r], n, mpix.MPI_BYTE, 1 - r, 3),
                       c.isend(src[r], n, mpix.MPI_BYTE, 1 - r, 3)]
            mpix.waitall(reqs[r])

        w.run_ranks(body)
        for r in range(2):
            assert torch.equal(dst[r].cpu(), src[1 - r].cpu())
        # a request can be waited once (proc_p2p.cpp:147: consumed)
        assert err(lambda: mpix.wait(reqs[0][0])) == "INVALID_REQUEST"
        assert err(lambda: mpix.wait(None)) == "INVALID_REQUEST"
        # a conventional request in an enqueue wait has no queue (Appendix A6)
        c0 = ctx[0].comm
        t = torch.zeros(4, dtype=torch.int32, device=0)
        r1 = w.comm(1).irecv(t, 4, mpix.MPI_INT, 0, 9)
        assert err(lambda: mpix.waitall_enqueue([r1])) == "STREAM_MISMATCH"
        w.comm(0).send(t, 4, mpix.MPI_INT, 1, 9)
        mpix.wait(r1)


def test_conventional_error_precedence_and_multiplex_rules():
    """rank -> count -> tag for conventional p2p (Appendix A5); MULTIPLEX_COMM
    for conventional calls on a multiplex comm; NOT_MULTIPLEX for stream calls
    on a single-stream comm; INVALID_INDEX / WILDCARD_DST."""
    with gpu_world(2) as (w, ctx):
        t = torch.zeros(16, dtype=torch.int32, device=0)
        wc = w.comm(0)
        assert err(lambda: wc.isend(t, -1, mpix.MPI_INT, 1, -1)) == "INVALID_COUNT"
        assert err(lambda: ctx[0].comm.isend_enqueue(t, -1, mpix.MPI_INT, 1, -1)) == "INVALID_TAG"
        assert err(lambda: wc.isend(t, 1, mpix.MPI_INT, 5, 0)) == "INVALID_RANK"
        mux = {}

        def mk(r):
            mux[r] = w.comm(r).stream_comm_create_multiplex(
                [mpix.Stream.from_cuda(mpix.testing.new_stream(0)) for _ in range(2)])

        w.run_ranks(mk)
        assert err(lambda: mux[0].isend(t, 1, mpix.MPI_INT, 1, 0)) == "MULTIPLEX_COMM"
        assert err(lambda: ctx[0].comm.stream_isend(t, 1, mpix.MPI_INT, 1, 0, 0, 0)) == "NOT_MULTIPLEX"
        assert err(lambda: mux[0].stream_isend(t, 1, mpix.MPI_INT, 1, 0, 2, 0)) == "INVALID_INDEX"
        assert err(lambda: mux[0].stream_isend(t, 1, mpix.MPI_INT, 1, 0, 0, 5)) == "INVALID_INDEX"
        assert err(lambda: mux[0].stream_irecv(t, 1, mpix.MPI_INT, 1, 0, 0,
                                               mpix.MPIX_ANY_INDEX)) == "WILDCARD_DST"


def test_multiplex_stream_p2p_indices_select_streams():
    """2 ranks x 2 local GPU streams: the same tag from (src_idx i) to
    (dst_idx j) for all four (i, j) pairs; each receive gets exactly its
    pair's payload (the indices are part of the match)."""
    n = 5000
    with gpu_world(2) as (w, ctx):
        mux, streams = {}, {}

        def mk(r):
            streams[r] = [mpix.testing.new_stream(0) for _ in range(2)]
            mux[r] = w.comm(r).stream_comm_create_multiplex(
                [mpix.Stream.from_cuda(s) for s in streams[r]])

        w.run_ranks(mk)
        src = {(i, j): rand_bytes(n, 100 + 2 * i + j) for i in range(2) for j in range(2)}
        dst = {(i, j): torch.zeros(n, dtype=torch.uint8, device=0) for i in range(2) for j in range(2)}
        torch.cuda.synchronize()

        def body(r):
            c = mux[r]
            if r == 0:
                reqs = [c.stream_isend(src[(i, j)], n, mpix.MPI_BYTE, 1, 4, i, j)
                        for i in range(2) for j in range(2)]
            else:
                reqs = [c.stream_irecv(dst[(i, j)], n, mpix.MPI_BYTE, 0, 4, i, j)
                        for j in range(2) for i in reversed(range(2))]
            mpix.waitall(reqs)

        w.run_ranks(body)
        for k in src:
            assert torch.equal(dst[k].cpu(), src[k].cpu()), k
        # blocking forms
        x, y = rand_bytes(777, 5), torch.zeros(777, dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        w.run_ranks(lambda r: mux[0].stream_send(x, 777, mpix.MPI_BYTE, 1, 6, 1, 0) if r == 0
                    else mux[1].stream_recv(y, 777, mpix.MPI_BYTE, 0, 6, 1, 0))
        assert torch.equal(x.cpu(), y.cpu())


def test_mixed_mode_conventional_send_to_recv_enqueue():
    """Appendix A7: rank 0's member of a stream comm passed STREAM_NULL (no
    enqueue there), its conventional MPI_Send matches rank 1's Recv_enqueue."""
    n = 70_000
    with gpu_world(2) as (w, ctx):
        comms = {}

        def mk(r):
            comms[r] = w.comm(r).stream_comm_create(None if r == 0 else ctx[1].mstream)

        w.run_ranks(mk)
        src = rand_bytes(n, 9)
        dst = torch.zeros(n, dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        assert err(lambda: comms[0].send_enqueue(src, n, mpix.MPI_BYTE, 1, 2)) == "NOT_ENQUEUE_COMM"

        def body(r):
            if r == 0:
                comms[0].send(src, n, mpix.MPI_BYTE, 1, 2)
            else:
                comms[1].recv_enqueue(dst, n, mpix.MPI_BYTE, 0, 2)

        w.run_ranks(body)
        sync_all(ctx)
        assert torch.equal(dst.cpu(), src.cpu())


def test_conventional_wildcard_receive_dynamic(monkeypatch):
    monkeypatch.setenv("MPIX_MATCHING", "dynamic")
    with gpu_world(3) as (w, ctx):
        x = {r: torch.full((4,), r, dtype=torch.int32, device=0) for r in (1, 2)}
        y = [torch.zeros(4, dtype=torch.int32, device=0) for _ in range(2)]
        torch.cuda.synchronize()

        def body(r):
            if r == 0:
                for k in range(2):
                    w.comm(0).recv(y[k], 4, mpix.MPI_INT, mpix.MPI_ANY_SOURCE, mpix.MPI_ANY_TAG)
            else:
                w.comm(r).send(x[r], 4, mpix.MPI_INT, 0, r)

        w.run_ranks(body)
        assert sorted(int(t[0]) for t in y) == [1, 2]


def test_conventional_and_multiplex_system_scope(monkeypatch):
    monkeypatch.setenv("MPIX_FORCE_SYS", "1")
    n = 300_000
    with gpu_world(2) as (w, ctx):
        mux = {}

        def mk(r):
            mux[r] = w.comm(r).stream_comm_create_multiplex(
                [mpix.Stream.from_cuda(mpix.testing.new_stream(0)) for _ in range(2)])

        w.run_ranks(mk)
        src = [rand_bytes(n, 40 + r) for r in range(2)]
        dst = [torch.zeros(n, dtype=torch.uint8, device=0) for _ in range(2)]
        dst2 = [torch.zeros(n, dtype=torch.uint8, device=0) for _ in range(2)]
        torch.cuda.synchronize()

        def body(r):
            c = w.comm(r)
            reqs = [c.irecv(dst[r], n, mpix.MPI_BYTE, 1 - r, 1), c.isend(src[r], n, mpix.MPI_BYTE, 1 - r, 1)]
            reqs += [mux[r].stream_irecv(dst2[r], n, mpix.MPI_BYTE, 1 - r, 2, 0, 1),
                     mux[r].stream_isend(src[r], n, mpix.MPI_BYTE, 1 - r, 2, 0, 1)]
            mpix.waitall(reqs)

        w.run_ranks(body)
        for r in range(2):
            assert torch.equal(dst[r].cpu(), src[1 - r].cpu())
            assert torch.equal(dst2[r].cpu(), src[1 - r].cpu())


@pytest.mark.parametrize("matching", ["static", "dynamic"])
def test_multiplex_indices_under_both_matching_modes(matching, monkeypatch):
    """The (src_idx, dst_idx) selection holds in both engines; MPIX_ANY_INDEX
    sources need the dynamic engine (UNSUPPORTED on a static comm)."""
    monkeypatch.setenv("MPIX_MATCHING", matching)
    n = 2048
    with gpu_world(2) as (w, ctx):
        mux = {}

        def mk(r):
            mux[r] = w.comm(r).stream_comm_create_multiplex(
                [mpix.Stream.from_cuda(mpix.testing.new_stream(0)) for _ in range(2)])

        w.run_ranks(mk)
        src = {(i, j): rand_bytes(n, 200 + 2 * i + j) for i in range(2) for j in range(2)}
        dst = {(i, j): torch.zeros(n, dtype=torch.uint8, device=0) for i in range(2) for j in range(2)}
        torch.cuda.synchronize()

        def body(r):
            c = mux[r]
            if r == 0:
                reqs = [c.stream_isend(src[(i, j)], n, mpix.MPI_BYTE, 1, 4, i, j)
                        for i in range(2) for j in range(2)]
            else:
                reqs = [c.stream_irecv(dst[(i, j)], n, mpix.MPI_BYTE, 0, 4, i, j)
                        for j in range(2) for i in reversed(range(2))]
            mpix.waitall(reqs)

        w.run_ranks(body)
        for k in src:
            assert torch.equal(dst[k].cpu(), src[k].cpu()), k
        t = torch.zeros(n, dtype=torch.uint8, device=0)
        if matching == "static":
            assert err(lambda: mux[1].stream_irecv(t, n, mpix.MPI_BYTE, 0, 4, mpix.MPIX_ANY_INDEX, 0)) \
                == "UNSUPPORTED"
            return
        # ANY_INDEX: two receives on dst_idx 0 take the sends from src_idx 1 and 0
        any_dst = [torch.zeros(n, dtype=torch.uint8, device=0) for _ in range(2)]
        torch.cuda.synchronize()

        def body2(r):
            c = mux[r]
            if r == 0:
                reqs = [c.stream_isend(src[(i, 0)], n, mpix.MPI_BYTE, 1, 5, i, 0) for i in (1, 0)]
            else:
                reqs = [c.stream_irecv(any_dst[k], n, mpix.MPI_BYTE, 0, 5, mpix.MPIX_ANY_INDEX, 0)
                        for k in range(2)]
            mpix.waitall(reqs)

        w.run_ranks(body2)
        got = sorted(bytes(x.cpu().numpy()[:4]) for x in any_dst)
        exp = sorted(bytes(src[(i, 0)].cpu().numpy()[:4]) for i in range(2))
        assert got == exp
