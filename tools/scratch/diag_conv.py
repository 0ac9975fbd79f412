import os, sys, time
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ["MPIX_SPIN_TIMEOUT_MS"] = "3000"
sys.path.insert(0, ".")
t0 = time.time()
import torch
torch.zeros(1, device=0)
print("cuda init", time.time() - t0, flush=True)
from paper_2208_13707_b200 import mpix
for n in (0, 8, 0):
    w = mpix.World(2, [0, 0])
    src = [torch.ones(max(n, 1), dtype=torch.uint8, device=0) for _ in range(2)]
    dst = [torch.zeros(max(n, 1), dtype=torch.uint8, device=0) for _ in range(2)]
    torch.cuda.synchronize()
    t = time.time()
    def body(r):
        c = w.comm(r)
        for _ in range(3):
            c.send(src[r], n, mpix.MPI_BYTE, 1 - r, 7)
            c.recv(dst[r], n, mpix.MPI_BYTE, 1 - r, 7)
    w.run_ranks(body)
    print("n", n, "time", time.time() - t, "errors", mpix.rank_error(0), mpix.rank_error(1), flush=True)
    t = time.time()
    w.finalize()
    print("finalize", time.time() - t, flush=True)
