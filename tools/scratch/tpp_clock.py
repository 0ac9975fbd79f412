import os, sys, statistics as st
os.environ["MPIX_TRACE"] = "1"
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, "/root/repo")
import torch
from paper_2208_13707_b200 import mpix
w = mpix.World(2, [0, 0]); ctx = {}
def setup(r):
    s = mpix.testing.new_stream(0); ctx[r] = (s, w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s)))
w.run_ranks(setup)
b0 = torch.zeros(16, dtype=torch.uint8, device=0); b1 = torch.zeros(16, dtype=torch.uint8, device=0)
d, h = mpix.testing.pingpong(ctx[0][1], ctx[1][1], b0, b1, 8, 400, ctx[0][0], ctx[1][0])
torch.cuda.synchronize()
A = sorted(mpix.trace_read(0, 4096), key=lambda r: r["seq"])
sends = [r for r in A if not r["is_recv"]][100:]
def c(r, k): return r["t"][k] if k < 6 else r["gt"][k - 5]
names = ["entry", "head stores", "warp0", "pre issued", "payload in regs", "scan done", "lane0 block", "ll_post", "fence.sc"]
print("half RTT us", d / 800 * 1e6)
for k in range(1, 9):
    print(f"{names[k-1]:>16s} -> {names[k]:16s} {st.median([c(r, k) - c(r, k - 1) for r in sends]):8.0f} cycles")
w.finalize()
