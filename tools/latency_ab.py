"""Small-message latency probe for A/B builds: native ping-pong (2 ranks,
GPU 0) and native loopback at 8 B / 4 KiB / 64 KiB."""
import os
import sys

sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch  # noqa: E402

from paper_2208_13707_b200 import mpix  # noqa: E402

w = mpix.World(2, [0, 0])
ctx = {}


def setup(r):
    s = mpix.testing.new_stream(0)
    ctx[r] = (s, w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s)))


w.run_ranks(setup)
pp, lb = {}, {}
big = torch.zeros(1 << 20, dtype=torch.uint8, device=0)
big2 = torch.zeros(1 << 20, dtype=torch.uint8, device=0)
for nb in (8, 4096, 65536):
    b0 = torch.zeros(max(nb, 16), dtype=torch.uint8, device=0)
    b1 = torch.zeros(max(nb, 16), dtype=torch.uint8, device=0)
    mpix.testing.pingpong(ctx[0][1], ctx[1][1], b0, b1, nb, 20, ctx[0][0], ctx[1][0])
    vals = []
    for _ in range(3):
        d, _ = mpix.testing.pingpong(ctx[0][1], ctx[1][1], b0, b1, nb, 500, ctx[0][0], ctx[1][0])
        vals.append(d / 1000 * 1e6)
    pp[nb] = round(sorted(vals)[1], 2)
    mpix.testing.loopback(ctx[0][1], big, big2, nb, 20, ctx[0][0])
    vals = []
    for _ in range(3):
        d, _ = mpix.testing.loopback(ctx[0][1], big, big2, nb, 500, ctx[0][0])
        vals.append(d / 500 * 1e6)
    lb[nb] = round(sorted(vals)[1], 2)
print("pingpong half RTT us", pp, "loopback us", lb)
for r in range(2):
    ctx[r][0].synchronize()
w.finalize()
