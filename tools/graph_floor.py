"""Launch floor inside a CUDA graph: G back-to-back empty kernels per graph."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_13707_b200 import mpix  # noqa: E402

mpix.lib()
s = mpix.testing.new_stream(0)
G, R = 64, 20
mpix.testing.graph_begin(s)
for _ in range(G):
    mpix.testing.empty(s)
g = mpix.testing.graph_end(s)
mpix.testing.graph_launch(g, s)
s.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(R):
    mpix.testing.graph_launch(g, s)
e1.record(s)
s.synchronize()
print(f"graph empty kernel: {e0.elapsed_time(e1) * 1e3 / (G * R):.2f} us/kernel")
