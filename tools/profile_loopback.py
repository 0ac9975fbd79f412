"""Minimal driver for ncu: the bench's N=1 step (256 MiB loopback
Isend/Irecv/Waitall_enqueue on one stream), W warm-up + K steps, nothing else.
k_p2p launches alternate send (index 2i) / receive (index 2i+1)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_13707_b200 import mpix  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=256 << 20)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--ranks", type=int, default=1)
ap.add_argument("--window", type=int, default=1)
a = ap.parse_args()
w = mpix.World(1, [0])
s = mpix.testing.new_stream(0)
c = w.comm(0).stream_comm_create(mpix.Stream.from_cuda(s))
src = torch.empty(a.size, dtype=torch.uint8, device=0)
dst = torch.zeros(a.size, dtype=torch.uint8, device=0)
mpix.testing.fill_pattern(src, a.size, 1, 0, s)
torch.cuda.synchronize()
for i in range(a.warmup + a.steps):
    reqs = []
    for k in range(a.window):  # window > 1: one coalesced k_batch per step
        reqs.append(c.isend_enqueue(src, a.size, mpix.MPI_BYTE, 0, k))
        reqs.append(c.irecv_enqueue(dst, a.size, mpix.MPI_BYTE, 0, k))
    mpix.waitall_enqueue(reqs)
torch.cuda.synchronize()
assert torch.equal(src, dst)
w.finalize()
print("ok")
