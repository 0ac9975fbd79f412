import os, sys
sys.path.insert(0, "/root/repo")
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch
from paper_2208_13707_b200 import mpix
w = mpix.World(2, [0, 0]); ctx = {}
def setup(r):
    s = mpix.testing.new_stream(0); ctx[r] = (s, w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s)))
w.run_ranks(setup)
for S in (1 << 20, 16 << 20, 256 << 20):
    xs = [torch.full((S,), r + 1, dtype=torch.uint8, device=0) for r in range(2)]
    xd = [torch.zeros(S, dtype=torch.uint8, device=0) for r in range(2)]
    torch.cuda.synchronize()
    X = (ctx[0][1], ctx[1][1], xs[0], xd[0], xs[1], xd[1], S)
    mpix.testing.exchange(*X, 3, ctx[0][0], ctx[1][0])
    K = 20
    t = mpix.testing.exchange(*X, K, ctx[0][0], ctx[1][0]) / K
    torch.cuda.synchronize()
    print(S, "step us", round(t * 1e6, 1), "HBM frac", round(4 * S / t / 1e9 / 6535, 3), int(xd[0][0]), int(xd[1][-1]))
w.finalize()
