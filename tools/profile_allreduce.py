"""Minimal ncu driver: Allreduce_enqueue of 256 MiB (bf16 by default) over P
ranks on GPU 0, W warm-up + K calls per rank."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_13707_b200 import mpix  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=2)
ap.add_argument("--bytes", type=int, default=256 << 20)
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--reduce-only", action="store_true",
                help="reduce stage alone for every rank in turn (ncu serialises kernels, so the\n"
                     "spinning entry/exit barriers of ranks sharing a GPU cannot be profiled)")
ap.add_argument("--oneshot", action="store_true")
a = ap.parse_args()
tdt, mdt = {"bf16": (torch.bfloat16, mpix.MPIX_BFLOAT16), "f32": (torch.float32, mpix.MPI_FLOAT)}[a.dtype]
cnt = a.bytes // torch.tensor([], dtype=tdt).element_size()
if a.reduce_only:
    s = mpix.testing.new_stream(0)
    sb = [torch.ones(cnt, dtype=tdt, device=0) for _ in range(a.P)]
    rb = [torch.empty(cnt, dtype=tdt, device=0) for _ in range(a.P)]
    for _ in range(a.iters):
        for me in range(a.P):
            mpix.testing.reduce_only(a.P, me, sb, rb, cnt, mdt, mpix.MPI_SUM, not a.oneshot, s)
    s.synchronize()
    assert float(rb[0][0]) == float(a.P)
    print("ok")
    sys.exit(0)
w = mpix.World(a.P, [0] * a.P)
ctx = {}


def setup(r):
    s = mpix.testing.new_stream(0)
    ctx[r] = (s, w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s)))


w.run_ranks(setup)
sb = [torch.ones(cnt, dtype=tdt, device=0) for _ in range(a.P)]
rb = [torch.empty(cnt, dtype=tdt, device=0) for _ in range(a.P)]
torch.cuda.synchronize()
w.run_ranks(lambda r: [ctx[r][1].allreduce_enqueue(sb[r], rb[r], cnt, mdt) for _ in range(a.iters)])
torch.cuda.synchronize()
assert float(rb[0][0]) == float(a.P)
w.finalize()
print("ok")
