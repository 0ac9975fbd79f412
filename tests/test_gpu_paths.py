"""GPU: the same parity checks with the runtime forced down each internal path
(inline 1-kernel ops vs proto+copy+fin, eager vs staged blocking sends, tiny
descriptor rings that force slot reuse). Knobs are read at MPIX_World_init."""
import os

import pytest
import torch

from paper_2208_13707_b200 import mpix
from tests.gpu_util import gpu_world, sync_all

pytestmark = pytest.mark.gpu

VARIANTS = {
    "all_split": {"MPIX_INLINE_BYTES": "0"},
    "all_inline": {"MPIX_INLINE_BYTES": str(1 << 30)},
    "tiny_eager": {"MPIX_EAGER_BYTES": "16"},
    "tiny_ring": {"MPIX_RING_SLOTS": "2"},
    "ring3_split": {"MPIX_RING_SLOTS": "3", "MPIX_INLINE_BYTES": "0", "MPIX_EAGER_BYTES": "0"},
    # the cross-GPU (system-scope) kernel instantiations, on one GPU
    "sys_scope": {"MPIX_FORCE_SYS": "1"},
    "sys_scope_split": {"MPIX_FORCE_SYS": "1", "MPIX_INLINE_BYTES": "0", "MPIX_RING_SLOTS": "4"},
    # the device matching engine (wildcard-capable) on concrete patterns
    "dynamic": {"MPIX_MATCHING": "dynamic"},
    "dynamic_split_sys": {"MPIX_MATCHING": "dynamic", "MPIX_INLINE_BYTES": "0",
                          "MPIX_RING_SLOTS": "4", "MPIX_FORCE_SYS": "1"},
    "dynamic_nobatch": {"MPIX_MATCHING": "dynamic", "MPIX_BATCH": "0", "MPIX_EAGER_BYTES": "16"},
}


@pytest.fixture(params=sorted(VARIANTS))
def variant(request, monkeypatch):
    for k, v in VARIANTS[request.param].items():
        monkeypatch.setenv(k, v)
    return request.param


def rb(n, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, 256, (max(n, 1),), dtype=torch.uint8, generator=g)[:n].to(0)


def test_variant_pingpong_and_loopback(variant):
    sizes = [0, 5, 16, 17, 4096, 70001, 1 << 20]
    with gpu_world(2) as (w, ctx):
        srcs = [rb(n, n + 1) for n in sizes]
        mids = [torch.zeros(max(n, 1), dtype=torch.uint8, device=0) for n in sizes]
        backs = [torch.zeros(max(n, 1), dtype=torch.uint8, device=0) for n in sizes]
        torch.cuda.synchronize()

        def rank(r):
            c = ctx[r].comm
            for i, n in enumerate(sizes):
                if r == 0:
                    c.send_enqueue(srcs[i], n, mpix.MPI_BYTE, 1, i)
                    c.recv_enqueue(backs[i], n, mpix.MPI_BYTE, 1, 100 + i)
                else:
                    c.recv_enqueue(mids[i], n, mpix.MPI_BYTE, 0, i)
                    c.send_enqueue(mids[i], n, mpix.MPI_BYTE, 0, 100 + i)

        w.run_ranks(rank)
        sync_all(ctx)
        for i, n in enumerate(sizes):
            assert torch.equal(backs[i][:n].cpu(), srcs[i].cpu()), (variant, n)


def test_variant_window_and_self(variant):
    with gpu_world(2) as (w, ctx):
        m = 24
        n = 3000
        src = torch.randint(0, 256, (m, n), dtype=torch.uint8, device=0)
        dst = torch.zeros_like(src)
        self_dst = torch.zeros_like(src)
        torch.cuda.synchronize()

        def rank(r):
            c = ctx[r].comm
            if r == 0:
                reqs = [c.isend_enqueue(src[i], n, mpix.MPI_BYTE, 1, i % 5) for i in range(m)]
                for i in range(m):  # self-messages through blocking calls
                    c.send_enqueue(src[i], n, mpix.MPI_BYTE, 0, 50)
                    c.recv_enqueue(self_dst[i], n, mpix.MPI_BYTE, 0, 50)
            else:
                reqs = [c.irecv_enqueue(dst[i], n, mpix.MPI_BYTE, 0, i % 5) for i in range(m)]
            mpix.waitall_enqueue(reqs)

        w.run_ranks(rank)
        sync_all(ctx)
        assert torch.equal(dst.cpu(), src.cpu())
        assert torch.equal(self_dst.cpu(), src.cpu())


def test_variant_allreduce(variant):
    from tests.test_gpu_allreduce import make_inputs, oracle
    P = 3
    for count in (3, 4096 + 1, 300001):
        with gpu_world(P) as (w, ctx):
            ins = make_inputs(P, count, "f32", seed=count)
            sb = [x.to(0) for x in ins]
            out = [torch.zeros_like(x) for x in sb]
            torch.cuda.synchronize()
            w.run_ranks(lambda r: ctx[r].comm.allreduce_enqueue(sb[r], out[r], count, mpix.MPI_FLOAT))
            sync_all(ctx)
            exp = oracle(ins, "f32", mpix.MPI_SUM)
            for r in range(P):
                assert torch.equal(out[r].cpu(), exp)
