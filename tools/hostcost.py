"""Host-side cost of the enqueue calls (Python ctypes -> C ABI -> launch)."""
import os, sys, time
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import torch
from paper_2208_13707_b200 import mpix
w = mpix.World(1, [0]); s = torch.cuda.Stream()
c = w.comm(0).stream_comm_create(mpix.Stream.from_cuda(s))
src = torch.ones(64, dtype=torch.uint8, device=0); dst = torch.zeros(64, dtype=torch.uint8, device=0)
L = mpix.lib(); h = c.h; ps, pd = src.data_ptr(), dst.data_ptr()
r1, r2 = C.c_uint64(), C.c_uint64()
arr = (C.c_uint64 * 2)()
N = 2000
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(N):
        L.MPIX_Isend_enqueue(ps, 8, 1, 0, 1, h, C.byref(r1))
        L.MPIX_Irecv_enqueue(pd, 8, 1, 0, 1, h, C.byref(r2))
        arr[0] = r1.value; arr[1] = r2.value
        L.MPIX_Waitall_enqueue(2, arr, None)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("host us per message (3 calls): %.2f   wall incl. GPU: %.2f" % ((t1 - t0) / N * 1e6, (t2 - t0) / N * 1e6))
t0 = time.perf_counter()
for i in range(N):
    mpix.testing.empty(s)
t1 = time.perf_counter(); torch.cuda.synchronize()
print("host us per empty-kernel launch via ctypes: %.2f" % ((t1 - t0) / N * 1e6))
t0 = time.perf_counter()
for i in range(N):
    L.MPIX_Type_size(1)
print("ctypes call floor us: %.2f" % ((time.perf_counter() - t0) / N * 1e6))
w.finalize()
