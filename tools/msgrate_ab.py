"""Message-rate probe for A/B builds (cfg4 shape: 8 ranks x 4 streams, window
64, 8-byte messages, native driver); matching mode from MPIX_MATCHING."""
import os
import sys

sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch  # noqa: E402

from paper_2208_13707_b200 import mpix  # noqa: E402
from paper_2208_13707_b200.workloads import msgrate  # noqa: E402

P, S, W, B = 8, 4, 64, 50
w = mpix.World(P, [0] * P)
ctxs = [[] for _ in range(P)]


def setup(r):
    for _ in range(S):
        s = mpix.testing.new_stream(0)
        ctxs[r].append((s, w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s))))


w.run_ranks(setup)
bufs = [[(torch.zeros(2, dtype=torch.int32, device=0),
          torch.zeros((W, 2), dtype=torch.int32, device=0)) for _ in range(S)] for r in range(P)]
msgrate(w, ctxs, S, W, 1, bufs)
rs = sorted(msgrate(w, ctxs, S, W, B, bufs)["msgs_per_s"] for _ in range(5))
torch.cuda.synchronize()
print(os.environ.get("MPIX_MATCHING", "static"), "M msgs/s", [round(x / 1e6, 2) for x in rs])
w.finalize()
