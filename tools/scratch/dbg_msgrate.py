"""Debug driver: cfg4 message-rate ring at small scale with a short watchdog.
python tools/dbg_msgrate.py P S W B"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MPIX_SPIN_TIMEOUT_MS", "3000")
import torch  # noqa: E402

from paper_2208_13707_b200 import mpix  # noqa: E402
from paper_2208_13707_b200.workloads import msgrate  # noqa: E402

P, S, W, B = (int(x) for x in sys.argv[1:5])
w = mpix.World(P, [0] * P)
ctxs = [[] for _ in range(P)]


def setup(r):
    for k in range(S):
        s = mpix.testing.new_stream(0)
        ctxs[r].append((s, w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s))))


w.run_ranks(setup)
bufs = [[(torch.tensor([r, k], dtype=torch.int32, device=0),
          torch.full((W, 2), -1, dtype=torch.int32, device=0)) for k in range(S)] for r in range(P)]
torch.cuda.synchronize()
l0 = mpix.launch_count()
res = msgrate(w, ctxs, S, W, B, bufs)
torch.cuda.synchronize()
print("launches", mpix.launch_count() - l0, res)
print("errors", [mpix.rank_error(r) for r in range(P)])
ok = True
for r in range(P):
    left = (r + P - 1) % P
    for k in range(S):
        rb = bufs[r][k][1].cpu()
        ok &= bool((rb[:, 0] == left).all()) and bool((rb[:, 1] == k).all())
print("payload ok", ok)
w.finalize()
