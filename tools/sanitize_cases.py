"""Small cases of the enqueue path for the sanitizers (tools/sanitize.sh).
--ranks 1: self-messages on one stream (every cross-CTA wait is inside one
launch, so it runs under compute-sanitizer's kernel serialisation);
--ranks 2: two ranks on GPU 0 driven by two host threads (ping-pong, windows,
conventional p2p, allreduce) — for ThreadSanitizer on the host runtime."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("MPIX_SPIN_TIMEOUT_MS", "20000")
import torch  # noqa: E402

from paper_2208_13707_b200 import mpix  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ranks", type=int, default=1)
a = ap.parse_args()
sizes = [0, 1, 8, 16, 17, 4096, 65536, 65537, 1 << 20]
P = a.ranks
w = mpix.World(P, [0] * P)
ctx = {}


def setup(r):
    s = mpix.testing.new_stream(0)
    ctx[r] = (s, w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s)))


w.run_ranks(setup)
nmax = max(sizes) + 64
src = [torch.arange(nmax, dtype=torch.int32, device=0).to(torch.uint8) + r for r in range(P)]
dst = [torch.zeros(nmax, dtype=torch.uint8, device=0) for _ in range(P)]
torch.cuda.synchronize()
bad = []


def body(r):
    s, c = ctx[r]
    peer = (r + 1) % P
    frm = (r - 1) % P
    for n in sizes:
        # non-blocking window: Isend + Irecv + Waitall
        q1 = c.isend_enqueue(src[r], n, mpix.MPI_BYTE, peer, 1)
        q2 = c.irecv_enqueue(dst[r], n, mpix.MPI_BYTE, frm, 1)
        mpix.waitall_enqueue([q1, q2])
        s.synchronize()
        if n and not torch.equal(dst[r][:n], src[frm][:n]):
            bad.append(("window", r, n))
        # blocking: send (eager or staged) then receive
        c.send_enqueue(src[r], n, mpix.MPI_BYTE, peer, 2)
        c.recv_enqueue(dst[r], n, mpix.MPI_BYTE, frm, 2)
        s.synchronize()
        if n and not torch.equal(dst[r][:n], src[frm][:n]):
            bad.append(("blocking", r, n))
    x = torch.full((4099,), float(r + 1), device=0)
    y = torch.zeros(4099, device=0)
    torch.cuda.synchronize()  # torch fills on its own stream; ours does not wait for it
    if P == 1 or mpix.device_coresident(0):
        c.allreduce_enqueue(x, y, 4099, mpix.MPI_FLOAT)
        s.synchronize()
        if float(y[0]) != sum(range(1, P + 1)):
            bad.append(("allreduce", r, float(y[0])))
    c.check()


w.run_ranks(body)
w.finalize()
print("sanitize cases:", "ok" if not bad else bad, "lib", mpix.LIB_PATH)
sys.exit(1 if bad else 0)
