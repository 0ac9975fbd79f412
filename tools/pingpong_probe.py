"""Native ping-pong half round trip (2 ranks on GPU 0), 8 B .. 64 KiB.
Run with MPIX_FORCE_SYS=1 to price the system-scope primitives cross-GPU
ranks use."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch  # noqa: E402

from paper_2208_13707_b200 import mpix  # noqa: E402

w = mpix.World(2, [0, 0])
ctx = {}


def setup(r):
    s = mpix.testing.new_stream(0)
    ctx[r] = (s, w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s)))


w.run_ranks(setup)
out = {}
for nb in (8, 4096, 65536, 1 << 20):
    b0 = torch.zeros(max(nb, 16), dtype=torch.uint8, device=0)
    b1 = torch.zeros(max(nb, 16), dtype=torch.uint8, device=0)
    mpix.testing.pingpong(ctx[0][1], ctx[1][1], b0, b1, nb, 20, ctx[0][0], ctx[1][0])
    d, h = mpix.testing.pingpong(ctx[0][1], ctx[1][1], b0, b1, nb, 500, ctx[0][0], ctx[1][0])
    out[nb] = round(d / 1000 * 1e6, 2)
print("force_sys" if os.environ.get("MPIX_FORCE_SYS") == "1" else "gpu-scope", "half RTT us", out)
for r in range(2):
    ctx[r][0].synchronize()
w.finalize()
