"""Per-call device-time breakdown of the loopback step (events between calls)."""
import os, sys
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2208_13707_b200 import mpix
S = int(sys.argv[1]) if len(sys.argv) > 1 else 256 << 20
w = mpix.World(1, [0]); s = torch.cuda.Stream()
c = w.comm(0).stream_comm_create(mpix.Stream.from_cuda(s))
src = torch.ones(S, dtype=torch.uint8, device=0); dst = torch.zeros(S, dtype=torch.uint8, device=0)
torch.cuda.synchronize()
N = 20
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(N)]
for it in range(3):
    r1 = c.isend_enqueue(src, S, 1, 0, 1); r2 = c.irecv_enqueue(dst, S, 1, 0, 1); mpix.waitall_enqueue([r1, r2])
torch.cuda.synchronize()
for i in range(N):
    ev[i][0].record(s)
    r1 = c.isend_enqueue(src, S, 1, 0, 1)
    ev[i][1].record(s)
    r2 = c.irecv_enqueue(dst, S, 1, 0, 1)
    ev[i][2].record(s)
    mpix.waitall_enqueue([r1, r2])
    ev[i][3].record(s)
torch.cuda.synchronize()
import statistics as st
parts = ["isend", "irecv", "waitall"]
for k in range(3):
    print(S, parts[k], "%.2f us" % st.median(ev[i][k].elapsed_time(ev[i][k + 1]) * 1e3 for i in range(N)))
print(S, "step", "%.2f us" % st.median(ev[i][0].elapsed_time(ev[i][3]) * 1e3 for i in range(N)))
# blocking self send/recv
for i in range(N):
    ev[i][0].record(s); c.send_enqueue(src, S, 1, 0, 2); ev[i][1].record(s); c.recv_enqueue(dst, S, 1, 0, 2); ev[i][2].record(s)
torch.cuda.synchronize()
print(S, "send(blocking,staged)", "%.2f us" % st.median(ev[i][0].elapsed_time(ev[i][1]) * 1e3 for i in range(N)))
print(S, "recv(blocking)", "%.2f us" % st.median(ev[i][1].elapsed_time(ev[i][2]) * 1e3 for i in range(N)))
assert torch.equal(src, dst)
w.finalize()
