"""cfg4 message rate alone (8 ranks x 4 streams, window 64), for host-path A/B."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch
from paper_2208_13707_b200 import mpix
from paper_2208_13707_b200.workloads import msgrate
P, S, W, B = 8, 4, 64, 50
w = mpix.World(P, [0] * P)
ctxs = [[] for _ in range(P)]
def setup(r):
    for k in range(S):
        s = mpix.testing.new_stream(0)
        ctxs[r].append((s, w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s))))
w.run_ranks(setup)
bufs = [[(torch.zeros(2, dtype=torch.int32, device=0), torch.zeros((W, 2), dtype=torch.int32, device=0)) for _ in range(S)] for r in range(P)]
msgrate(w, ctxs, S, W, 1, bufs)
for _ in range(2):
    msgrate(w, ctxs, S, W, B, bufs)
res = [msgrate(w, ctxs, S, W, B, bufs) for _ in range(3)]
print("msgs/s M", [round(r["msgs_per_s"] / 1e6, 2) for r in res], "enqueue_s", [round(r["enqueue_s"] * 1e3, 2) for r in res])
w.finalize()
