"""GPU: the BASELINE.json configs at their real sizes, checked against the
oracle.

- cfg3: MPIX_Allreduce_enqueue sum of 256 MiB per rank, fp32 (67,108,864
  elements) and bf16 (134,217,728), P = 2 / 4 / 8, both value sets ("exact"
  and the order-sensitive uniform(-1,1)), between a producer kernel and a
  consumer (checksum) kernel on the rank's stream. Bit-exact against the
  rank-ordered fold (oracle/streamix_oracle.c orc_allreduce_gen, the same fold
  as orc_allreduce_f32/bf16, pinned to the reference-composed allreduce in
  tests/golden/allreduce.json): the device checksum of every rank's output
  equals the oracle's checksum of the full output, and sampled elements are
  equal bit for bit. Inputs are generated on the device (MPIXT_Fill_values)
  and on the host (orc_value_f32/bf16) from the same hash; the input
  checksum is compared too.
- cfg1: 2 ranks, Send_enqueue/Recv_enqueue ping-pong of the 1 MiB fp32
  buffer x[i] = float(i % 1024) * 0.5, 200 round trips: the FNV-1a-64 of both
  ranks' buffers equals the reference's own (tests/golden/cfg1.json, produced
  by oracle/_ref running the unmodified reference).
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2208_13707_b200 import mpix
from tests.gpu_util import gpu_world

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MiB = 1 << 20
DT = {"f32": (torch.float32, mpix.MPI_FLOAT, 4, np.float32),
      "bf16": (torch.bfloat16, mpix.MPIX_BFLOAT16, 2, np.uint16)}


def dev_checksum(buf, nbytes, stream):
    out = torch.zeros(1, dtype=torch.int64, device=buf.device)
    mpix.testing.checksum(buf, nbytes, out, stream)
    stream.synchronize()
    return int(out.item()) & (2**64 - 1)


def samples(count, k=64, seed=0):
    rng = np.random.default_rng(seed)
    idx = np.concatenate([[0, 1, count // 2, count - 2, count - 1], rng.integers(0, count, k)])
    return np.unique(idx).astype(np.uint64)


def run_cfg3(P, dt, value_set, in_place=False):
    tdt, mdt, es, npdt = DT[dt]
    count = 256 * MiB // es
    with gpu_world(P) as (w, ctx):
        sb = [torch.empty(count, dtype=tdt, device=0) for _ in range(P)]
        rb = sb if in_place else [torch.empty(count, dtype=tdt, device=0) for _ in range(P)]
        for r in range(P):  # producer kernel on the rank's stream
            mpix.testing.fill_values(sb[r], count, mdt, value_set, r, ctx[r].stream)
        assert dev_checksum(sb[P - 1], 256 * MiB, ctx[P - 1].stream) == \
            O.gen_checksum(P - 1, count, dt, value_set)
        w.run_ranks(lambda r: ctx[r].comm.allreduce_enqueue(sb[r], rb[r], count, mdt))
        idx = samples(count, seed=P * 10 + value_set)
        exp_cs, exp_s = O.allreduce_gen(P, count, dt, value_set, 1, idx)
        ti = torch.from_numpy(idx.astype(np.int64)).to(0)
        for r in range(P):  # consumer kernel on the rank's stream
            assert dev_checksum(rb[r], 256 * MiB, ctx[r].stream) == exp_cs, f"rank {r}"
            got = rb[r][ti].cpu()
            got = got.view(torch.int16).numpy().view(np.uint16) if dt == "bf16" else got.numpy()
            assert np.array_equal(got.view(np.uint8), exp_s.view(np.uint8)), f"rank {r} samples"


@pytest.mark.parametrize("value_set", [0, 1], ids=["exact", "uniform"])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_cfg3_allreduce_256MiB_bit_exact(P, dt, value_set):
    run_cfg3(P, dt, value_set)


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_cfg3_allreduce_256MiB_in_place_P8(dt):
    run_cfg3(8, dt, 1, in_place=True)


def test_cfg1_pingpong_matches_reference_fnv():
    g = json.load(open(os.path.join(GOLD, "cfg1.json")))
    n, iters = g["count"], g["iters"]
    x = (torch.arange(n, dtype=torch.int64) % 1024).to(torch.float32) * 0.5
    with gpu_world(2) as (w, ctx):
        xs = x.to(0)
        back = torch.zeros(n, dtype=torch.float32, device=0)
        mid = torch.zeros(n, dtype=torch.float32, device=0)
        torch.cuda.synchronize()

        def body(r):
            c = ctx[r].comm
            for _ in range(iters):
                if r == 0:
                    c.send_enqueue(xs, n, mpix.MPI_FLOAT, 1, 0)
                    c.recv_enqueue(back, n, mpix.MPI_FLOAT, 1, 1)
                else:
                    c.recv_enqueue(mid, n, mpix.MPI_FLOAT, 0, 0)
                    c.send_enqueue(mid, n, mpix.MPI_FLOAT, 0, 1)

        w.run_ranks(body)
        for c in ctx:
            c.stream.synchronize()
        assert O.fnv1a64(back.cpu().numpy()) == g["fnv1a64_rank0"]
        assert O.fnv1a64(mid.cpu().numpy()) == g["fnv1a64_rank1"]
