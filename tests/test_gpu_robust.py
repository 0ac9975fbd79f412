"""GPU: failure reporting and progress guarantees.

- A device watchdog expiry is a STICKY error (MPIX_ERR_TIMEOUT) that every
  later call naming the rank returns, including host waits and
  MPIX_Comm_check. The reference reports every failure through Result<Err>
  (proj/include/streamix/result.hpp:36-45); a kernel that gives up a flag
  wait must not leave garbage behind MPI_SUCCESS.
- Held (batched) non-blocking operations progress without a later ordering
  call on their stream: the reference registers I-operations at once
  (proj/src/proc_enqueue.cpp:67-114).
- Conventional waits return the matched message's status (source, tag,
  stream index, bytes, truncated), as Proc::wait does
  (proj/src/proc_p2p.cpp:146-156, deliver at proj/src/endpoint.cpp:17-24).
- MPI_Comm_free refuses while a conventional receive is undelivered
  (PENDING_OPS, proj/src/proc_comm.cpp:182-184).
"""
import contextlib
import os
import time

import pytest
import torch

from paper_2208_13707_b200 import mpix
from tests.gpu_util import gpu_world

pytestmark = pytest.mark.gpu


def err(fn):
    try:
        fn()
        return "OK"
    except mpix.MPIXError as e:
        return e.name


@contextlib.contextmanager
def env(**kv):
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update({k: str(v) for k, v in kv.items()})
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def world_with_comms(P):
    w = mpix.World(P, [0] * P)
    ctx = {}

    def setup(r):
        s = mpix.testing.new_stream(0)
        ctx[r] = (s, w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s)))

    w.run_ranks(setup)
    return w, ctx


def test_watchdog_expiry_is_sticky_on_every_call():
    """A blocking self-receive with no send (Appendix A13: blocks forever in
    the reference) trips the 300 ms watchdog; from then on every call of the
    rank returns TIMEOUT instead of MPI_SUCCESS."""
    with env(MPIX_SPIN_TIMEOUT_MS=300):
        w, ctx = world_with_comms(1)
    try:
        s, c = ctx[0]
        buf = torch.zeros(64, dtype=torch.uint8, device=0)
        c.recv_enqueue(buf, 64, mpix.MPI_BYTE, 0, 5)
        t0 = time.time()
        s.synchronize()
        assert time.time() - t0 < 10
        assert mpix.rank_error(0) == 2  # ERRW_WAIT_DONE
        assert err(c.check) == "TIMEOUT"
        assert err(lambda: c.isend_enqueue(buf, 8, mpix.MPI_BYTE, 0, 1)) == "TIMEOUT"
        assert err(lambda: c.recv_enqueue(buf, 8, mpix.MPI_BYTE, 0, 1)) == "TIMEOUT"
        assert err(lambda: c.allreduce_enqueue(buf, buf, 2, mpix.MPI_INT)) == "TIMEOUT"
        assert err(lambda: w.comm(0).send(buf, 8, mpix.MPI_BYTE, 0, 1)) == "TIMEOUT"
        assert err(lambda: w.comm(0).isend(buf, 8, mpix.MPI_BYTE, 0, 1)) == "TIMEOUT"
    finally:
        torch.cuda.synchronize()
        w.finalize()


def test_host_wait_returns_timeout_not_success():
    """MPI_Wait on a receive that never matches: the device wait gives up at
    the watchdog and the host call reports it."""
    with env(MPIX_SPIN_TIMEOUT_MS=300):
        w = mpix.World(1, [0])
    try:
        buf = torch.zeros(16, dtype=torch.int32, device=0)
        r = w.comm(0).irecv(buf, 16, mpix.MPI_INT, 0, 77)
        assert err(lambda: mpix.wait(r)) == "TIMEOUT"
    finally:
        torch.cuda.synchronize()
        w.finalize()


def test_allreduce_with_an_absent_member_times_out_cleanly():
    """Rank 1 never enters: rank 0's fused allreduce kernel gives up at its
    entry barrier and the failure is visible on rank 0 only."""
    with env(MPIX_SPIN_TIMEOUT_MS=300):
        w, ctx = world_with_comms(2)
    try:
        x = torch.ones(1024, dtype=torch.float32, device=0)
        y = torch.zeros(1024, dtype=torch.float32, device=0)
        ctx[0][1].allreduce_enqueue(x, y, 1024, mpix.MPI_FLOAT)
        ctx[0][0].synchronize()
        assert err(ctx[0][1].check) == "TIMEOUT"
        assert err(ctx[1][1].check) == "OK"
    finally:
        torch.cuda.synchronize()
        w.finalize()


@pytest.mark.parametrize("n", [8, 4096, 1 << 20, 8 << 20])
def test_held_isend_progresses_without_an_ordering_call(n):
    """Isend_enqueue on rank 0's stream is held in its batch; rank 1's
    blocking Recv_enqueue on another stream is synchronised by the host
    before rank 0 makes any further call. The flusher launches the held
    batch, so the receive completes (the reference registers I-operations at
    once, proc_enqueue.cpp:67-114)."""
    with gpu_world(2) as (w, ctx):
        src = torch.randint(0, 256, (n,), dtype=torch.uint8, device=0)
        dst = torch.zeros(n, dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        r = ctx[0].comm.isend_enqueue(src, n, mpix.MPI_BYTE, 1, 4)
        ctx[1].comm.recv_enqueue(dst, n, mpix.MPI_BYTE, 0, 4)
        t0 = time.time()
        ctx[1].stream.synchronize()
        assert time.time() - t0 < 5
        assert torch.equal(dst, src)
        mpix.wait_enqueue(r)


def test_held_irecv_progresses_for_a_host_waited_sender():
    """The mirror case: rank 1's Irecv_enqueue is held in its batch; rank 0
    sends on the same comm with a conventional MPI_Isend (it publishes its
    buffer, zero copy) and blocks in MPI_Wait on the host — which completes
    only once the held receive has run and pulled the payload."""
    n = 3 << 20
    with gpu_world(2) as (w, ctx):
        src = torch.randint(0, 256, (n,), dtype=torch.uint8, device=0)
        dst = torch.zeros(n, dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        r = ctx[1].comm.irecv_enqueue(dst, n, mpix.MPI_BYTE, 0, 9)
        t0 = time.time()
        st = mpix.wait(ctx[0].comm.isend(src, n, mpix.MPI_BYTE, 1, 9))
        assert time.time() - t0 < 5 and st["bytes"] == n
        mpix.wait_enqueue(r)
        ctx[1].stream.synchronize()
        assert torch.equal(dst, src)


@pytest.mark.parametrize("n,cap", [(1000, 600), (300, 600), (0, 16), (3 << 20, 1 << 20),
                                   (200_000, 200_000)])
def test_conventional_statuses_are_the_matched_message(n, cap):
    """MPI_Recv / MPI_Wait statuses: source, tag, bytes = min(len, cap),
    truncated = len > cap (endpoint.cpp:17-24); a send's status is
    (me, tag, bytes) (proc_p2p.cpp:54-58)."""
    with gpu_world(2) as (w, ctx):
        src = torch.randint(0, 256, (max(n, 1),), dtype=torch.uint8, device=0)
        dst = torch.zeros(max(cap, 1), dtype=torch.uint8, device=0)
        dst2 = torch.zeros(max(cap, 1), dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        out = {}

        def body(r):
            c = w.comm(r)
            if r == 0:
                c.send(src, n, mpix.MPI_BYTE, 1, 11)
                out["s"] = mpix.wait(c.isend(src, n, mpix.MPI_BYTE, 1, 12))
            else:
                out["r1"] = c.recv(dst, cap, mpix.MPI_BYTE, 0, 11)
                out["r2"] = mpix.waitall([c.irecv(dst2, cap, mpix.MPI_BYTE, 0, 12)])[0]

        w.run_ranks(body)
        k = min(n, cap)
        for key, tag in (("r1", 11), ("r2", 12)):
            st = out[key]
            assert st == {"source": 0, "tag": tag, "source_index": -2, "bytes": k,
                          "truncated": n > cap}, (key, st)
        assert torch.equal(dst[:k], src[:k]) and torch.equal(dst2[:k], src[:k])
        assert out["s"] == {"source": 0, "tag": 12, "source_index": -2, "bytes": n,
                            "truncated": False}


def test_wildcard_statuses_name_the_sender():
    """Dynamic matching: ANY_SOURCE / ANY_TAG receives report which message
    they took (the reference's deliver fills source and tag)."""
    with env(MPIX_MATCHING="dynamic"):
        w = mpix.World(3, [0, 0, 0])
    try:
        bufs = {r: torch.full((4096 * r,), r, dtype=torch.uint8, device=0) for r in (1, 2)}
        dst = [torch.zeros(8192, dtype=torch.uint8, device=0) for _ in range(2)]
        torch.cuda.synchronize()
        out = {}

        def body(r):
            c = w.comm(r)
            if r == 0:
                reqs = [c.irecv(dst[i], 8192, mpix.MPI_BYTE, mpix.MPI_ANY_SOURCE, mpix.MPI_ANY_TAG)
                        for i in range(2)]
                out[0] = mpix.waitall(reqs)
            else:
                c.send(bufs[r], 4096 * r, mpix.MPI_BYTE, 0, 40 + r)

        w.run_ranks(body)
        seen = set()
        for i, st in enumerate(out[0]):
            src = st["source"]
            assert src in (1, 2) and st["tag"] == 40 + src and st["bytes"] == 4096 * src
            assert not st["truncated"]
            assert int(dst[i][0]) == src and int(dst[i][st["bytes"] - 1]) == src
            seen.add(src)
        assert seen == {1, 2}
    finally:
        torch.cuda.synchronize()
        w.finalize()


def test_multiplex_status_carries_the_source_index():
    with gpu_world(2) as (w, ctx):
        mux = {}

        def mk(r):
            mux[r] = w.comm(r).stream_comm_create_multiplex(
                [mpix.Stream.from_cuda(mpix.testing.new_stream(0)) for _ in range(2)])

        w.run_ranks(mk)
        src = torch.arange(64, dtype=torch.int32, device=0)
        dst = torch.zeros(64, dtype=torch.int32, device=0)
        torch.cuda.synchronize()
        out = {}

        def body(r):
            if r == 0:
                mux[0].stream_send(src, 64, mpix.MPI_INT, 1, 3, 1, 0)
            else:
                out[1] = mux[1].stream_recv(dst, 64, mpix.MPI_INT, 0, 3, 1, 0)

        w.run_ranks(body)
        assert out[1] == {"source": 0, "tag": 3, "source_index": 1, "bytes": 256, "truncated": False}
        assert torch.equal(dst, src)
        w.run_ranks(lambda r: mux[r].free())


def test_comm_free_refuses_while_a_conventional_receive_is_pending():
    with gpu_world(2) as (w, ctx):
        comms = {}
        w.run_ranks(lambda r: comms.__setitem__(r, w.comm(r).stream_comm_create(
            mpix.Stream.from_cuda(mpix.testing.new_stream(0)))))
        buf = torch.zeros(4, dtype=torch.int32, device=0)
        src = torch.arange(4, dtype=torch.int32, device=0)
        torch.cuda.synchronize()
        r = comms[1].irecv(buf, 4, mpix.MPI_INT, 0, 3)
        assert err(comms[1].free) == "PENDING_OPS"
        comms[0].send(src, 4, mpix.MPI_INT, 1, 3)
        assert mpix.wait(r)["bytes"] == 16
        w.run_ranks(lambda q: comms[q].free())
        assert torch.equal(buf, src)


def test_destroyed_stream_hint_is_bad_hint():
    """A cudaStream_t hint naming a stream destroyed through this library is
    BAD_HINT without dereferencing the handle — the reference's live-queue
    registry (proj/src/exec_queue.cpp:100-103, checked at
    proj/src/proc_stream.cpp:17); a live one is accepted."""
    h = mpix.C.c_void_p()
    assert mpix.lib().MPIXT_Stream_create(0, mpix.C.byref(h)) == 0
    live = h.value

    def hint(v):
        info = mpix.Info()
        info.set("type", "cudaStream_t")
        info.set_hex("value", v.to_bytes(8, "little"))
        return err(lambda: mpix.Stream(info).free())

    with gpu_world(1):
        assert hint(live) == "OK"
        assert mpix.lib().MPIXT_Stream_destroy(mpix.C.c_void_p(live)) == 0
        assert hint(live) == "BAD_HINT"
