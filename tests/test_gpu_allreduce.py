"""GPU parity of MPIX_Allreduce_enqueue.

Oracle: element-wise left fold in rank order 0..P-1 (fp32 accumulator, one
final RNE rounding for bf16, wrapping int32). Both kernels compute each
element with one thread in that order, so results must be bit-exact.
"""
import numpy as np
import pytest
import torch

from paper_2208_13707_b200 import mpix
from tests.gpu_util import gpu_world, sync_all

pytestmark = pytest.mark.gpu

DT = {
    "f32": (torch.float32, mpix.MPI_FLOAT),
    "bf16": (torch.bfloat16, mpix.MPIX_BFLOAT16),
    "i32": (torch.int32, mpix.MPI_INT),
    "f64": (torch.float64, mpix.MPI_DOUBLE),
}


def make_inputs(P, count, dt, seed):
    g = torch.Generator().manual_seed(seed)
    out = []
    for r in range(P):
        if dt == "i32":
            t = torch.randint(-2**31, 2**31 - 1, (count,), dtype=torch.int64, generator=g).to(torch.int32)
        else:
            t = (torch.rand(count, generator=g, dtype=torch.float64) * 2 - 1).to(DT[dt][0])
        out.append(t)
    return out


def oracle(inputs, dt, op):
    if dt == "i32":
        acc = inputs[0].numpy().astype(np.int64)
        for x in inputs[1:]:
            xv = x.numpy().astype(np.int64)
            if op == mpix.MPI_SUM:
                acc = acc + xv
            elif op == mpix.MPI_MAX:
                acc = np.where(xv > acc, xv, acc)
            else:
                acc = np.where(xv < acc, xv, acc)
        return torch.from_numpy(((acc + 2**31) % 2**32 - 2**31).astype(np.int32))
    accdt = np.float64 if dt == "f64" else np.float32
    acc = inputs[0].to(torch.float64 if dt == "f64" else torch.float32).numpy().astype(accdt)
    for x in inputs[1:]:
        xv = x.to(torch.float64 if dt == "f64" else torch.float32).numpy().astype(accdt)
        if op == mpix.MPI_SUM:
            acc = (acc + xv).astype(accdt)
        elif op == mpix.MPI_MAX:
            acc = np.where(xv > acc, xv, acc)
        else:
            acc = np.where(xv < acc, xv, acc)
    return torch.from_numpy(acc).to(DT[dt][0])


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("dt", ["f32", "bf16", "i32", "f64"])
@pytest.mark.parametrize("count", [1, 7, 1000, 65536 + 5, 1 << 20])
def test_allreduce_sum_bit_exact(P, dt, count):
    with gpu_world(P) as (w, ctx):
        ins = make_inputs(P, count, dt, seed=P * 1000 + count)
        sb = [x.to(0) for x in ins]
        rb = [torch.zeros_like(x) for x in sb]
        torch.cuda.synchronize()

        def rank(r):
            ctx[r].comm.allreduce_enqueue(sb[r], rb[r], count, DT[dt][1], mpix.MPI_SUM)

        w.run_ranks(rank)
        sync_all(ctx)
        exp = oracle(ins, dt, mpix.MPI_SUM)
        for r in range(P):
            got = rb[r].cpu()
            assert torch.equal(got.view(torch.uint8) if False else got, exp), (r, (got != exp).sum())


@pytest.mark.parametrize("op", [mpix.MPI_MAX, mpix.MPI_MIN])
@pytest.mark.parametrize("dt", ["f32", "i32", "bf16"])
def test_allreduce_max_min(op, dt):
    P, count = 4, 50001
    with gpu_world(P) as (w, ctx):
        ins = make_inputs(P, count, dt, seed=7)
        sb = [x.to(0) for x in ins]
        rb = [torch.zeros_like(x) for x in sb]
        torch.cuda.synchronize()
        w.run_ranks(lambda r: ctx[r].comm.allreduce_enqueue(sb[r], rb[r], count, DT[dt][1], op))
        sync_all(ctx)
        exp = oracle(ins, dt, op)
        for r in range(P):
            assert torch.equal(rb[r].cpu(), exp)


@pytest.mark.parametrize("P", [2, 4])
def test_allreduce_in_place_and_repeated(P):
    count = 300000
    with gpu_world(P) as (w, ctx):
        ins = make_inputs(P, count, "f32", seed=11)
        bufs = [x.to(0).clone() for x in ins]
        torch.cuda.synchronize()
        w.run_ranks(lambda r: ctx[r].comm.allreduce_enqueue("in_place", bufs[r], count, mpix.MPI_FLOAT))
        sync_all(ctx)
        exp = oracle(ins, "f32", mpix.MPI_SUM)
        for r in range(P):
            assert torch.equal(bufs[r].cpu(), exp)
        # a second round on the result (epochs advance, flags are monotone)
        w.run_ranks(lambda r: ctx[r].comm.allreduce_enqueue("in_place", bufs[r], count, mpix.MPI_FLOAT))
        sync_all(ctx)
        exp2 = oracle([exp] * P, "f32", mpix.MPI_SUM)
        for r in range(P):
            assert torch.equal(bufs[r].cpu(), exp2)


def test_allreduce_unaligned_buffers():
    P, count = 3, 12345
    with gpu_world(P) as (w, ctx):
        ins = make_inputs(P, count, "f32", seed=3)
        big = [torch.zeros(count + 1, dtype=torch.float32, device=0) for _ in range(P)]
        for r in range(P):
            big[r][1:] = ins[r].to(0)
        rb = [torch.zeros(count + 3, dtype=torch.float32, device=0) for _ in range(P)]
        torch.cuda.synchronize()
        w.run_ranks(lambda r: ctx[r].comm.allreduce_enqueue(big[r][1:], rb[r][3:], count, mpix.MPI_FLOAT))
        sync_all(ctx)
        exp = oracle(ins, "f32", mpix.MPI_SUM)
        for r in range(P):
            assert torch.equal(rb[r][3:].cpu(), exp)


@pytest.mark.parametrize("twoshot", [False, True])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_reduce_stage_alone_matches_oracle(dt, twoshot):
    """MPIXT_Reduce_only (the profiling entry: reduce stage without the
    barriers) computes the same bits as the full collective's oracle."""
    P, count = 4, (1 << 18) + 37
    ins = make_inputs(P, count, dt, 11)
    exp = oracle(ins, dt, mpix.MPI_SUM)
    sb = [x.to(0) for x in ins]
    rb = [torch.zeros(count, dtype=DT[dt][0], device=0) for _ in range(P)]
    s = mpix.testing.new_stream(0)
    for me in range(P):
        mpix.testing.reduce_only(P, me, sb, rb, count, DT[dt][1], mpix.MPI_SUM, twoshot, s)
    s.synchronize()
    for r in range(P):
        assert torch.equal(rb[r].cpu().view(torch.int16 if dt == "bf16" else torch.int32),
                           exp.view(torch.int16 if dt == "bf16" else torch.int32)), r


@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("case", ["plain", "in_place", "unaligned", "max_i32"])
def test_fused_single_launch_allreduce(P, case, monkeypatch):
    """The single-CTA allreduce (entry + two-shot chunk + exit in one launch),
    forced up to large counts, bit-exact with the rank-ordered oracle."""
    monkeypatch.setenv("MPIX_ALLREDUCE_ONESHOT_MAX", str(64 << 20))
    count = 300001
    dt = "i32" if case == "max_i32" else "f32"
    op = mpix.MPI_MAX if case == "max_i32" else mpix.MPI_SUM
    with gpu_world(P) as (w, ctx):
        ins = make_inputs(P, count, dt, seed=P + 17)
        off = 1 if case == "unaligned" else 0
        sb = [torch.zeros(count + off, dtype=DT[dt][0], device=0) for _ in range(P)]
        for r in range(P):
            sb[r][off:] = ins[r].to(0)
        rb = [torch.zeros(count + 2 * off, dtype=DT[dt][0], device=0) for _ in range(P)]
        torch.cuda.synchronize()
        l0 = mpix.launch_count()

        def body(r):
            if case == "in_place":
                ctx[r].comm.allreduce_enqueue("in_place", sb[r], count, DT[dt][1], op)
            else:
                ctx[r].comm.allreduce_enqueue(sb[r][off:], rb[r][2 * off:], count, DT[dt][1], op)

        w.run_ranks(body)
        launches = mpix.launch_count() - l0
        sync_all(ctx)
        exp = oracle(ins, dt, op)
        for r in range(P):
            got = sb[r].cpu() if case == "in_place" else rb[r][2 * off:].cpu()
            assert torch.equal(got, exp), r
        assert launches == P  # one launch per rank
