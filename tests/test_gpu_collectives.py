"""GPU parity of the enqueued collectives beyond Allreduce (
SURVEY.md §8(f) item 3): Reduce, Reduce_scatter_block, Bcast, Allgather and
Barrier, all in-stream between producer and consumer work.

Oracle: folds are the rank-ordered fold of tests/test_gpu_allreduce.oracle
(fp32 accumulator, one RNE rounding for bf16, wrapping int32) — the same
restatement as orc_allreduce_* in oracle/streamix_oracle.c — so results are
bit-exact; copies are byte-exact.
"""
import pytest
import torch

from paper_2208_13707_b200 import mpix
from tests.gpu_util import gpu_world, sync_all
from tests.test_gpu_allreduce import DT, make_inputs, oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("dt", ["f32", "bf16", "i32"])
@pytest.mark.parametrize("count", [5, 70001])
def test_reduce_to_root(P, dt, count):
    root = P - 1
    with gpu_world(P) as (w, ctx):
        ins = make_inputs(P, count, dt, seed=P * 7 + count)
        sb = [x.to(0) for x in ins]
        rb = [torch.full((count,), 3, dtype=DT[dt][0], device=0) for _ in range(P)]
        torch.cuda.synchronize()
        w.run_ranks(lambda r: ctx[r].comm.reduce_enqueue(sb[r], rb[r], count, DT[dt][1],
                                                         mpix.MPI_SUM, root))
        sync_all(ctx)
        assert torch.equal(rb[root].cpu(), oracle(ins, dt, mpix.MPI_SUM))
        for r in range(P):
            if r != root:  # untouched elsewhere
                assert bool((rb[r] == 3).all())


def test_reduce_in_place_at_root_and_max():
    P, count = 4, 12345
    with gpu_world(P) as (w, ctx):
        ins = make_inputs(P, count, "f32", seed=5)
        bufs = [x.to(0).clone() for x in ins]
        torch.cuda.synchronize()

        def body(r):
            c = ctx[r].comm
            if r == 0:
                c.reduce_enqueue("in_place", bufs[0], count, mpix.MPI_FLOAT, mpix.MPI_MAX, 0)
            else:
                c.reduce_enqueue(bufs[r], None, count, mpix.MPI_FLOAT, mpix.MPI_MAX, 0)

        w.run_ranks(body)
        sync_all(ctx)
        assert torch.equal(bufs[0].cpu(), oracle(ins, "f32", mpix.MPI_MAX))


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("dt", ["f32", "bf16", "i32", "f64"])
@pytest.mark.parametrize("rc", [1, 33333])
def test_reduce_scatter_block(P, dt, rc):
    with gpu_world(P) as (w, ctx):
        ins = make_inputs(P, P * rc, dt, seed=P + rc)
        sb = [x.to(0) for x in ins]
        rb = [torch.zeros(rc, dtype=DT[dt][0], device=0) for _ in range(P)]
        torch.cuda.synchronize()
        w.run_ranks(lambda r: ctx[r].comm.reduce_scatter_block_enqueue(sb[r], rb[r], rc, DT[dt][1]))
        sync_all(ctx)
        full = oracle(ins, dt, mpix.MPI_SUM)
        for r in range(P):
            assert torch.equal(rb[r].cpu(), full[r * rc:(r + 1) * rc]), r


@pytest.mark.parametrize("P", [2, 5, 8])
@pytest.mark.parametrize("n", [1, 4099, (3 << 20) + 7])
def test_bcast(P, n):
    root = 1
    with gpu_world(P) as (w, ctx):
        g = torch.Generator().manual_seed(n)
        data = torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g)
        bufs = [data.to(0) if r == root else torch.zeros(n, dtype=torch.uint8, device=0)
                for r in range(P)]
        torch.cuda.synchronize()
        w.run_ranks(lambda r: ctx[r].comm.bcast_enqueue(bufs[r], n, mpix.MPI_BYTE, root))
        sync_all(ctx)
        for r in range(P):
            assert torch.equal(bufs[r].cpu(), data), r


@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("n", [3, 65536 + 9])
@pytest.mark.parametrize("in_place", [False, True])
def test_allgather(P, n, in_place):
    with gpu_world(P) as (w, ctx):
        blocks = [torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int64,
                                generator=torch.Generator().manual_seed(r)).to(torch.int32)
                  for r in range(P)]
        sb = [b.to(0) for b in blocks]
        rb = [torch.zeros(P * n, dtype=torch.int32, device=0) for _ in range(P)]
        if in_place:
            for r in range(P):
                rb[r][r * n:(r + 1) * n] = sb[r]
        torch.cuda.synchronize()
        w.run_ranks(lambda r: ctx[r].comm.allgather_enqueue("in_place" if in_place else sb[r], rb[r],
                                                            n, mpix.MPI_INT))
        sync_all(ctx)
        exp = torch.cat(blocks)
        for r in range(P):
            assert torch.equal(rb[r].cpu(), exp), r


@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("nb", [12, 4096, (1 << 20) + 4], ids=["12B", "4KiB", "1MiB+4"])
def test_alltoall(P, nb):
    """Block q of rank r's sendbuf lands in block r of rank q's recvbuf, byte-exact
    (blocks of any size, including ones that are not multiples of 16 B)."""
    with gpu_world(P) as (w, ctx):
        src = [torch.randint(0, 256, (P * nb,), dtype=torch.uint8,
                             generator=torch.Generator().manual_seed(40 + r)) for r in range(P)]
        sb = [x.to(0) for x in src]
        rb = [torch.zeros(P * nb, dtype=torch.uint8, device=0) for _ in range(P)]
        torch.cuda.synchronize()
        for _ in range(2):  # twice: the epoch and the op records are reused correctly
            w.run_ranks(lambda r: ctx[r].comm.alltoall_enqueue(sb[r], rb[r], nb, mpix.MPI_BYTE))
        sync_all(ctx)
        for q in range(P):
            exp = torch.cat([src[r][q * nb:(q + 1) * nb] for r in range(P)])
            assert torch.equal(rb[q].cpu(), exp), q


def test_alltoall_errors():
    with gpu_world(2) as (w, ctx):
        x = torch.zeros(64, dtype=torch.int32, device=0)
        codes = {}

        def body(r):
            c = ctx[r].comm
            out = []
            for fn in (lambda: mpix.lib().MPIX_Alltoall_enqueue(1, 8, mpix.MPI_INT, x.data_ptr(), 8,
                                                                mpix.MPI_INT, c.h),
                       lambda: mpix.lib().MPIX_Alltoall_enqueue(x.data_ptr(), 8, mpix.MPI_INT,
                                                                x.data_ptr() + 256, 4,
                                                                mpix.MPI_INT, c.h)):
                out.append(mpix.error_string(fn()))
            codes[r] = out

        w.run_ranks(body)
        assert codes[0] == ["INVALID_ARG", "INVALID_COUNT"], codes


def test_barrier_orders_streams():
    """Rank 0 delays, then writes; Barrier_enqueue on every rank; every rank
    then reads rank 0's buffer through a Bcast: the write is visible."""
    P = 4
    with gpu_world(P) as (w, ctx):
        x = [torch.zeros(1024, dtype=torch.int32, device=0) for _ in range(P)]
        torch.cuda.synchronize()

        def body(r):
            c = ctx[r].comm
            for it in range(3):
                if r == 0:
                    mpix.testing.delay(200_000, ctx[0].stream)
                    with torch.cuda.stream(ctx[0].stream):
                        x[0].fill_(it + 1)
                c.barrier_enqueue()
                c.bcast_enqueue(x[r], 1024, mpix.MPI_INT, 0)
                c.barrier_enqueue()

        w.run_ranks(body)
        sync_all(ctx)
        for r in range(P):
            assert bool((x[r] == 3).all()), r


def test_collectives_error_codes():
    with gpu_world(2) as (w, ctx):
        c = ctx[0].comm
        t = torch.zeros(8, dtype=torch.float32, device=0)
        with pytest.raises(mpix.MPIXError) as e:
            c.bcast_enqueue(t, 8, mpix.MPI_FLOAT, 2)
        assert e.value.name == "INVALID_RANK"
        with pytest.raises(mpix.MPIXError) as e:
            c.reduce_enqueue(t, t, -1, mpix.MPI_FLOAT)
        assert e.value.name == "INVALID_COUNT"
        with pytest.raises(mpix.MPIXError) as e:
            w.comm(0).barrier_enqueue()
        assert e.value.name == "NOT_ENQUEUE_COMM"


def test_collectives_system_scope(monkeypatch):
    """The cross-GPU (system-scope) kernel instantiations, on one GPU
    (MPIX_FORCE_SYS=1): every collective once, bit-exact."""
    monkeypatch.setenv("MPIX_FORCE_SYS", "1")
    P, rc = 4, 4097
    with gpu_world(P) as (w, ctx):
        ins = make_inputs(P, P * rc, "bf16", seed=99)
        sb = [x.to(0) for x in ins]
        red = [torch.zeros(P * rc, dtype=torch.bfloat16, device=0) for _ in range(P)]
        rsb = [torch.zeros(rc, dtype=torch.bfloat16, device=0) for _ in range(P)]
        bc = [sb[r].clone() for r in range(P)]
        ag = [torch.zeros(P * P * rc, dtype=torch.bfloat16, device=0) for _ in range(P)]
        torch.cuda.synchronize()

        def body(r):
            c = ctx[r].comm
            c.reduce_enqueue(sb[r], red[r], P * rc, mpix.MPIX_BFLOAT16, mpix.MPI_SUM, 2)
            c.reduce_scatter_block_enqueue(sb[r], rsb[r], rc, mpix.MPIX_BFLOAT16)
            c.bcast_enqueue(bc[r], P * rc, mpix.MPIX_BFLOAT16, 3)
            c.allgather_enqueue(sb[r], ag[r], P * rc, mpix.MPIX_BFLOAT16)
            c.barrier_enqueue()

        w.run_ranks(body)
        sync_all(ctx)
        full = oracle(ins, "bf16", mpix.MPI_SUM)
        assert torch.equal(red[2].cpu(), full)
        for r in range(P):
            assert torch.equal(rsb[r].cpu(), full[r * rc:(r + 1) * rc])
            assert torch.equal(bc[r].cpu(), ins[3])
            assert torch.equal(ag[r].cpu(), torch.cat(ins))


@pytest.mark.parametrize("P", [2, 4, 8])
def test_reduce_scatter_block_in_place(P):
    rc = 10007
    with gpu_world(P) as (w, ctx):
        ins = make_inputs(P, P * rc, "f32", seed=P + 3)
        bufs = [x.to(0).clone() for x in ins]
        torch.cuda.synchronize()
        w.run_ranks(lambda r: ctx[r].comm.reduce_scatter_block_enqueue("in_place", bufs[r], rc,
                                                                       mpix.MPI_FLOAT))
        sync_all(ctx)
        full = oracle(ins, "f32", mpix.MPI_SUM)
        for r in range(P):
            assert torch.equal(bufs[r][:rc].cpu(), full[r * rc:(r + 1) * rc]), r
