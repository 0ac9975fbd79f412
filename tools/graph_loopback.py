"""8-byte self-message loopback captured in a CUDA graph (G iterations per
graph): per-iteration device time, optionally eager too (for ncu launch lists)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_13707_b200 import mpix  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--G", type=int, default=64)
ap.add_argument("--replays", type=int, default=10)
ap.add_argument("--size", type=int, default=8)
ap.add_argument("--graph", type=int, default=1, help="mpix_graph hint (1: graph-capturable comm)")
ap.add_argument("--eager", action="store_true", help="enqueue eagerly instead of replaying")
a = ap.parse_args()

w = mpix.World(1, [0])
st = {}


def body(r):
    s = mpix.testing.new_stream(0)
    c = w.comm(0).stream_comm_create(mpix.Stream.from_cuda(s, mpix_graph=str(a.graph)))
    x = torch.zeros(max(a.size, 16), dtype=torch.uint8, device=0)
    y = torch.zeros(max(a.size, 16), dtype=torch.uint8, device=0)

    def it(k):
        for _ in range(k):
            rq = [c.isend_enqueue(x, a.size, mpix.MPI_BYTE, 0, 1),
                  c.irecv_enqueue(y, a.size, mpix.MPI_BYTE, 0, 1)]
            mpix.waitall_enqueue(rq)

    it(8)
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if a.eager:
        e0.record(s)
        it(a.G * a.replays)
        e1.record(s)
    else:
        mpix.testing.graph_begin(s)
        it(a.G)
        g = mpix.testing.graph_end(s)
        mpix.testing.graph_launch(g, s)
        s.synchronize()
        e0.record(s)
        for _ in range(a.replays):
            mpix.testing.graph_launch(g, s)
        e1.record(s)
    s.synchronize()
    st["us"] = e0.elapsed_time(e1) * 1e3 / (a.G * a.replays)
    c.free()


w.run_ranks(body)
print(f"{'eager' if a.eager else 'graph'} size={a.size} graph_comm={a.graph}: {st['us']:.2f} us/iteration")
w.finalize()
