"""Probe: the symmetric heap across processes (torchrun --nproc-per-node 2).
Each rank writes its rank into its slice; every rank then reads every slice
through the shared virtual addresses."""
import ctypes as C
import os
import socket
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from paper_2208_13707_b200 import mpix

rank, n = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
dev = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
L = mpix.lib()
U64 = C.c_uint64
L.MPIX_Heap_create.argtypes = [C.c_int, C.c_int, C.c_int, U64, U64, C.POINTER(U64), C.POINTER(U64), C.POINTER(C.c_int)]
L.MPIX_Heap_attach.argtypes = [C.c_int, C.c_int]
base, slice_, fd = U64(), U64(), C.c_int()
L.MPIX_Heap_destroy.argtypes = []
ok_all = False
for k in range(16):
    cand = 0x600000000000 + (k << 40)
    rc = L.MPIX_Heap_create(rank, n, dev, 64 << 20, cand, C.byref(base), C.byref(slice_), C.byref(fd))
    flag = torch.tensor([1 if rc == 0 else 0])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    print("rank", rank, "candidate", hex(cand), "rc", rc, "all", int(flag[0]), flush=True)
    if int(flag[0]):
        ok_all = True
        break
    if rc == 0:
        L.MPIX_Heap_destroy()
assert ok_all
# exchange fds over unix sockets
path = f"/tmp/mpix_heap_probe_{os.environ.get('MASTER_PORT','0')}_{rank}"
srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
if os.path.exists(path):
    os.unlink(path)
srv.bind(path)
srv.listen(n)
dist.barrier()
for q in range(n):
    if q == rank:
        continue
    c = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    c.connect(f"/tmp/mpix_heap_probe_{os.environ.get('MASTER_PORT','0')}_{q}")
    socket.send_fds(c, [rank.to_bytes(4, "little")], [fd.value])
    c.close()
for _ in range(n - 1):
    conn, _ = srv.accept()
    msg, fds, _, _ = socket.recv_fds(conn, 4, 1)
    q = int.from_bytes(msg, "little")
    rc = L.MPIX_Heap_attach(q, fds[0])
    print("rank", rank, "attach", q, rc, flush=True)
    conn.close()
dist.barrier()
mine = base.value + slice_.value * rank
t = torch.full((1024,), rank + 1, dtype=torch.int32, device=dev)
C.CDLL("libcudart.so", mode=C.RTLD_GLOBAL) if False else None
import ctypes.util
cudart = torch.cuda.cudart()
torch.cuda.synchronize()
# write my slice with cudaMemcpy via torch: wrap raw pointer
class Raw:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (ptr, False), "version": 3}
view = torch.as_tensor(Raw(mine, 1024), device=f"cuda:{dev}")
view.copy_(t)
torch.cuda.synchronize()
dist.barrier()
ok = True
for q in range(n):
    v = torch.as_tensor(Raw(base.value + slice_.value * q, 1024), device=f"cuda:{dev}")
    val = int(v[0])
    ok &= val == q + 1
    print("rank", rank, "reads slice", q, "=", val, flush=True)
dist.barrier()
print("rank", rank, "OK" if ok else "FAIL", flush=True)
os.unlink(path)
dist.destroy_process_group()
