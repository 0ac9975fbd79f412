"""Driver for ncu: blocking 8-byte self Send_enqueue + Recv_enqueue on one
stream (one k_batch_tiny each: an LL post, then a polling receive that finds
it) — the handshake kernels of the ping-pong, runnable under ncu's kernel
serialisation."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch  # noqa: E402

from paper_2208_13707_b200 import mpix  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = mpix.World(1, [0])
s = mpix.testing.new_stream(0)
c = w.comm(0).stream_comm_create(mpix.Stream.from_cuda(s))
a = torch.arange(max(n, 16), dtype=torch.uint8, device=0)
b = torch.zeros(max(n, 16), dtype=torch.uint8, device=0)
torch.cuda.synchronize()
for i in range(iters):
    c.send_enqueue(a, n, mpix.MPI_BYTE, 0, 3)
    c.recv_enqueue(b, n, mpix.MPI_BYTE, 0, 3)
s.synchronize()
assert torch.equal(a[:n], b[:n])
w.finalize()
print("ok")
