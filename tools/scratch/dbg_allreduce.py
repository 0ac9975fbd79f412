import os, sys, time, struct
os.environ["MPIX_SPIN_TIMEOUT_MS"] = "2000"
sys.path.insert(0, "/root/repo")
import torch
from paper_2208_13707_b200 import mpix
from tests.gpu_util import gpu_world, sync_all
R = mpix.config()["ring_slots"]
def coll(comm, P):
    raw = comm.region_bytes()
    off = 2 * P * R * 64 + 2 * P * R * 8
    return [struct.unpack_from("<QQQQ", raw, off + 32 * q) for q in range(P)], [struct.unpack_from("<Q", raw, off + 32 * P + 8 * q)[0] for q in range(P)]
for P, count in [(1, 1), (2, 1), (2, 1)]:
    with gpu_world(P) as (w, ctx):
        sb = [torch.full((count,), float(r + 1), device=0) for r in range(P)]
        rb = [torch.zeros(count, device=0) for r in range(P)]
        torch.cuda.synchronize()
        print("streams", [c.stream.cuda_stream for c in ctx], "sb", [hex(x.data_ptr()) for x in sb], "rb", [hex(x.data_ptr()) for x in rb])
        t0 = time.time()
        w.run_ranks(lambda r: ctx[r].comm.allreduce_enqueue(sb[r], rb[r], count, mpix.MPI_FLOAT))
        sync_all(ctx)
        print(P, count, "t", round(time.time() - t0, 3), [float(x[0]) for x in rb], [mpix.rank_error(r) for r in range(P)], flush=True)
        for r in range(P):
            print("  rank", r, coll(ctx[r].comm, P))
