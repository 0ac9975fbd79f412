"""The small-message protocol: flag-in-data (LL) sends of
<= 12 bytes, polling blocking receives, host-paired small self-messages, and
held conventional operations. Every case is checked byte-exact against the
oracle pattern and, where the reference reports one, against its status
(deliver: bytes = min(len, cap), truncated = len > cap, endpoint.cpp:17-24)."""
import threading
import time

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2208_13707_b200 import mpix
from tests.gpu_util import gpu_world

LL_SIZES = [0, 1, 3, 4, 5, 8, 11, 12, 13, 16, 17]


def pattern(n, seed):
    return torch.from_numpy(O.fill_pattern(max(n, 1), seed, 1)[:max(n, 1)].copy()).to(0)


@pytest.mark.gpu
@pytest.mark.parametrize("n", LL_SIZES)
@pytest.mark.parametrize("order", ["send_first", "recv_first"])
def test_ll_sizes_blocking_and_nonblocking(n, order):
    """Blocking Send_enqueue + blocking Recv_enqueue, and Isend/Irecv +
    Waitall, across the 12-byte LL boundary, with the receive posted before or
    after the send (the LL post, the polling receive, the Dekker race with an
    Irecv posted first)."""
    with gpu_world(2) as (w, ctx):
        src = pattern(n, 11)
        d1 = torch.zeros(max(n, 1), dtype=torch.uint8, device=0)
        d2 = torch.zeros(max(n, 1), dtype=torch.uint8, device=0)
        torch.cuda.synchronize()

        def body(r):
            c = ctx[r].comm
            if r == 0:
                if order == "recv_first":
                    time.sleep(0.002)
                c.send_enqueue(src, n, mpix.MPI_BYTE, 1, 5)
                q = c.isend_enqueue(src, n, mpix.MPI_BYTE, 1, 6)
                mpix.waitall_enqueue([q])
            else:
                if order == "send_first":
                    time.sleep(0.002)
                q = c.irecv_enqueue(d2, n, mpix.MPI_BYTE, 0, 6)
                c.recv_enqueue(d1, n, mpix.MPI_BYTE, 0, 5)
                mpix.waitall_enqueue([q])

        w.run_ranks(body)
        for c in ctx:
            c.stream.synchronize()
        if n:
            assert torch.equal(d1[:n], src[:n]) and torch.equal(d2[:n], src[:n])


@pytest.mark.gpu
@pytest.mark.parametrize("n,cap", [(12, 4), (8, 8), (5, 100), (12, 1 << 17)])
def test_ll_truncation_and_status(n, cap):
    """An LL message into a smaller, equal, larger and non-inline (capacity
    above MPIX_INLINE_BYTES: the op-record path) receive buffer: bytes
    delivered and the status the reference reports."""
    with gpu_world(2) as (w, ctx):
        src = pattern(n, 3)
        dst = torch.zeros(cap, dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        out = {}

        def body(r):
            c = ctx[r].world_comm
            if r == 0:
                c.send(src, n, mpix.MPI_BYTE, 1, 7)
            else:
                out["st"] = c.recv(dst, cap, mpix.MPI_BYTE, 0, 7)

        w.run_ranks(body)
        k = min(n, cap)
        assert torch.equal(dst[:k].cpu(), src[:k].cpu())
        if cap > n:
            assert int(dst[k:].count_nonzero()) == 0
        st = out["st"]
        assert st["bytes"] == k and st["truncated"] == (n > cap)
        assert st["source"] == 0 and st["tag"] == 7


@pytest.mark.gpu
def test_ll_window_many_tags_out_of_order():
    """A window of 64 LL Isends over 8 tags, received in reverse tag order by
    Irecvs posted before and after: static matching by (tag, sequence)."""
    n, W, T = 8, 64, 8
    with gpu_world(2) as (w, ctx):
        src = torch.stack([pattern(n, 100 + i) for i in range(W)])
        dst = torch.zeros((W, n), dtype=torch.uint8, device=0)
        torch.cuda.synchronize()

        def body(r):
            c = ctx[r].comm
            if r == 0:
                qs = [c.isend_enqueue(src[i], n, mpix.MPI_BYTE, 1, i % T) for i in range(W)]
            else:
                order = sorted(range(W), key=lambda i: (-(i % T), i))
                qs = [c.irecv_enqueue(dst[i], n, mpix.MPI_BYTE, 0, i % T) for i in order]
            mpix.waitall_enqueue(qs)

        w.run_ranks(body)
        for c in ctx:
            c.stream.synchronize()
        assert torch.equal(dst, src)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 8, 12, 13, 4096, 65536])
def test_small_self_messages_host_paired(n):
    """Isend + Irecv to self in one batch (paired on the host: one copy, no
    descriptors), then the reverse order, then a held Isend whose Irecv comes
    in a later batch (not paired: the two-sided protocol)."""
    with gpu_world(1) as (w, ctx):
        c = ctx[0].comm
        src = pattern(n, 21)
        outs = [torch.zeros(max(n, 1), dtype=torch.uint8, device=0) for _ in range(3)]
        torch.cuda.synchronize()
        q1 = c.isend_enqueue(src, n, mpix.MPI_BYTE, 0, 1)
        q2 = c.irecv_enqueue(outs[0], n, mpix.MPI_BYTE, 0, 1)
        mpix.waitall_enqueue([q1, q2])
        q3 = c.irecv_enqueue(outs[1], n, mpix.MPI_BYTE, 0, 2)
        q4 = c.isend_enqueue(src, n, mpix.MPI_BYTE, 0, 2)
        mpix.waitall_enqueue([q3, q4])
        q5 = c.isend_enqueue(src, n, mpix.MPI_BYTE, 0, 3)
        q6 = c.irecv_enqueue(outs[2], n, mpix.MPI_BYTE, 0, 3)
        mpix.waitall_enqueue([q5, q6])
        ctx[0].stream.synchronize()
        for o in outs:
            if n:
                assert torch.equal(o[:n], src[:n])


@pytest.mark.gpu
def test_held_conventional_isend_progresses():
    """A conventional MPI_Isend joins its comm's batch (MPIX_CONV_BATCH): the
    sender makes no further call while the peer blocks in MPI_Recv; the
    flusher launches the held send."""
    n = 8
    with gpu_world(2) as (w, ctx):
        src = pattern(n, 5)
        dst = torch.zeros(n, dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        done = threading.Event()
        out = {}

        def body(r):
            c = ctx[r].world_comm
            if r == 0:
                out["q"] = c.isend(src, n, mpix.MPI_BYTE, 1, 3)
                done.wait(10)
                mpix.wait(out["q"])
            else:
                t0 = time.time()
                c.recv(dst, n, mpix.MPI_BYTE, 0, 3)
                out["t"] = time.time() - t0
                done.set()

        w.run_ranks(body)
        assert torch.equal(dst, src)
        assert out["t"] < 5


@pytest.mark.gpu
@pytest.mark.parametrize("n", [8, 4096])
def test_graph_comm_device_matched_self_messages_and_fallback(n):
    """Graph-capturable comm (sequences in device counters): a self Isend +
    Irecv in one launch are matched on the device (the receive copies, the
    send stands down). An earlier unmatched Isend on the same tag puts the
    send and receive counters out of step, so the next launch's host-expected
    pair does not match on the device and both take the two-sided protocol:
    the receive gets the earlier send, as static matching requires."""
    w = mpix.World(1, [0])
    try:
        s = mpix.testing.new_stream(0)
        c = w.comm(0).stream_comm_create(mpix.Stream.from_cuda(s, mpix_graph="1"))
        A, B, C = pattern(n, 31), pattern(n, 32), pattern(n, 33)
        X, Y, Z = [torch.zeros(n, dtype=torch.uint8, device=0) for _ in range(3)]
        tmp = torch.zeros(16, dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        # matched pair in one launch
        q1 = c.isend_enqueue(C, n, mpix.MPI_BYTE, 0, 4)
        q2 = c.irecv_enqueue(Z, n, mpix.MPI_BYTE, 0, 4)
        mpix.waitall_enqueue([q1, q2])
        # an unmatched Isend on tag 5, launched (a blocking self send/recv on
        # another tag closes the batches)
        qa = c.isend_enqueue(A, n, mpix.MPI_BYTE, 0, 5)
        c.send_enqueue(tmp, 8, mpix.MPI_BYTE, 0, 99)
        c.recv_enqueue(tmp, 8, mpix.MPI_BYTE, 0, 99)
        # host-expected pair, counters out of step: the receive takes A
        qb = c.isend_enqueue(B, n, mpix.MPI_BYTE, 0, 5)
        qx = c.irecv_enqueue(X, n, mpix.MPI_BYTE, 0, 5)
        mpix.waitall_enqueue([qx])
        qy = c.irecv_enqueue(Y, n, mpix.MPI_BYTE, 0, 5)
        mpix.waitall_enqueue([qa, qb, qy])
        s.synchronize()
        assert torch.equal(Z, C)
        assert torch.equal(X, A) and torch.equal(Y, B)
        assert mpix.rank_error(0) == 0
    finally:
        torch.cuda.synchronize()
        w.finalize()
