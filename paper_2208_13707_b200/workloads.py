"""Applications written against the enqueue API, used by the tests and
bench.py (BASELINE.json configs 4 and 5):

- `HaloStencil`: 3-D 7-point stencil on a 2x2x2 periodic decomposition. Each
  step packs the 6 faces, exchanges them with Isend/Irecv_enqueue +
  Waitall_enqueue, unpacks into the halos and runs the stencil, all in the
  rank's CUDA stream (no host synchronisation between steps). Pipelined
  (default): the interior [2, n-1]^3, which reads no halo, runs on a second
  stream while the faces are in flight; the boundary shell runs after the
  unpack.
- `fig3`: the reference's lock-regime message-rate bench (paper Fig. 3,
  proj/src/bench.cpp:118-235) over conventional p2p on GPU buffers: 2 ranks x
  T host threads, each pair on its own communicator, under one of the three
  host exclusion regimes (global lock / per communicator / serial context).
- `msgrate`: S single-stream comms per rank (the reference rejects enqueue on
  multiplex comms, proc_enqueue.cpp:24), ring neighbours, W outstanding
  8-byte Isend/Irecv_enqueue per stream, Waitall_enqueue per batch.

Both mirror the structure of the reference's own CPU driver for the same
workloads (oracle/ref_driver.cpp) and of PAPER.md Listing 2.
"""
from __future__ import annotations

from . import mpix

# face d: 0=-x 1=+x 2=-y 3=+y 4=-z 5=+z
OPP = [1, 0, 3, 2, 5, 4]


def coords(rank: int):
    return rank & 1, (rank >> 1) & 1, (rank >> 2) & 1


def neighbour(rank: int, d: int) -> int:
    """Rank of the neighbour across face d in the 2x2x2 periodic grid."""
    c = list(coords(rank))
    axis = d >> 1
    c[axis] = (c[axis] + (1 if d & 1 else -1)) % 2
    return c[0] | (c[1] << 1) | (c[2] << 2)


class HaloStencil:
    """One rank's block: (n+2)^3 fp32 with a one-cell halo, x fastest."""

    W0, W1 = 0.5, 1.0 / 12.0

    def __init__(self, rank: int, n: int, stream, comm, device=0, torch=None, pipelined=True):
        import torch as _t
        self.t = torch or _t
        self.pipelined = pipelined
        self.s2 = mpix.testing.new_stream(device) if pipelined else None
        self.rank, self.n, self.stream, self.comm = rank, n, stream, comm
        shape = ((n + 2) * (n + 2) * (n + 2),)
        self.u = self.t.zeros(shape, dtype=self.t.float32, device=device)
        self.v = self.t.zeros(shape, dtype=self.t.float32, device=device)
        self.sbuf = [self.t.zeros(n * n, dtype=self.t.float32, device=device) for _ in range(6)]
        self.rbuf = [self.t.zeros(n * n, dtype=self.t.float32, device=device) for _ in range(6)]

    def exchange(self):
        n, s = self.n, self.stream
        mpix.testing.halo_pack6(self.u, n, n, n, self.sbuf, s)
        reqs = []
        for d in range(6):  # halo d is filled by the neighbour across d, which sent its OPP(d) face
            reqs.append(self.comm.irecv_enqueue(self.rbuf[d], n * n, mpix.MPI_FLOAT,
                                                neighbour(self.rank, d), OPP[d]))
        for d in range(6):
            reqs.append(self.comm.isend_enqueue(self.sbuf[d], n * n, mpix.MPI_FLOAT,
                                                neighbour(self.rank, d), d))
        mpix.waitall_enqueue(reqs)
        mpix.testing.halo_unpack6(self.u, n, n, n, self.rbuf, s)

    def step(self):
        n = self.n
        if not self.pipelined:
            self.exchange()
            mpix.testing.stencil7(self.u, self.v, n, n, n, self.W0, self.W1, self.stream)
        else:
            ea = self.t.cuda.Event()
            ea.record(self.stream)
            self.s2.wait_event(ea)
            mpix.testing.stencil7_box(self.u, self.v, n, n, n, (2, n - 1) * 3, self.W0, self.W1,
                                      self.s2)
            eb = self.t.cuda.Event()
            eb.record(self.s2)
            self.exchange()
            mpix.testing.stencil7_shell(self.u, self.v, n, n, n, self.W0, self.W1, self.stream)
            self.stream.wait_event(eb)
        self.u, self.v = self.v, self.u


def msgrate(world, ctxs, S: int, W: int, batches: int, bufs) -> dict:
    """ctxs[r][k] = (torch stream, comm) for stream k of rank r; bufs[r][k] =
    (8-byte send buffer, W x 8-byte receive buffer). One native host thread
    per rank drives the C ABI (csrc/mpix_drivers.cpp, the analogue of the
    reference's C++ bench driver). Returns messages, host and device-timed
    seconds, and msgs/s over the larger of the two."""
    P = len(ctxs)
    comms, streams, sb, rb, devs = [], [], [], [], []
    for r in range(P):
        devs.append(ctxs[r][0][0].device.index or 0)
        for k in range(S):
            s, c = ctxs[r][k][0], ctxs[r][k][1]
            comms.append(c)
            streams.append(s)
            sb.append(bufs[r][k][0])
            rb.append(bufs[r][k][1])
    return mpix.testing.msgrate(comms, streams, sb, rb, devs, P, S, W, batches)


REGIMES = {0: "global", 1: "pervci", 2: "stream"}  # the reference's mode names (bench.cpp:102-108)


def fig3(T: int, W: int = 64, batches: int = 100, nbytes: int = 8, regime: int = 1,
         device: int = 0, torch=None) -> dict:
    """Paper Fig. 3 on the GPU path: regime 0 ("global") runs every p2p call
    under one process-wide lock with one internal stream per rank; 1
    ("pervci", the reference's per_vci_implicit) a lock and an internal stream
    per communicator; 2 ("stream", stream_explicit) gives each thread an
    explicit MPIX stream whose communicator is a lock-free serial context.
    Comms for regimes 0/1 are created on MPIX_STREAM_NULL, as the reference
    does (bench.cpp:157-171). Driven by native threads (MPIXT_Fig3)."""
    if torch is None:
        import torch
    w = mpix.World(2, [device, device])
    try:
        mpix.testing.set_exclusion(regime)
        comms = {0: [], 1: []}
        streams = {0: [], 1: []}

        def setup(r):
            for _ in range(T):
                st = mpix.Stream() if regime == 2 else None
                streams[r].append(st)
                comms[r].append(w.comm(r).stream_comm_create(st))

        w.run_ranks(setup)
        slot = max(nbytes, 1)
        bufs = [torch.zeros(slot * W + 1, dtype=torch.uint8, device=device) for _ in range(2 * T)]
        out = mpix.testing.fig3(comms[0] + comms[1], bufs, [device, device], T, W, batches, nbytes)
        out["regime"] = REGIMES[regime]

        def teardown(r):
            for c in comms[r]:
                c.free()
            for st in streams[r]:
                if st is not None:
                    st.free()

        w.run_ranks(teardown)
        return out
    finally:
        w.finalize()


def graph_latency(G: int = 64, R: int = 20) -> dict:
    """Latency-bound patterns enqueued eagerly vs captured into a CUDA graph
    (DESIGN.md §3b). G iterations are enqueued (or captured once and replayed),
    R times. Device time comes from CUDA events on each rank's stream, taking
    the max over ranks. Graph-capturable comms are used for both arms, so the
    kernels are the same and only the host launch path differs.
    - loopback_8B: Isend + Irecv + Waitall_enqueue of an 8-byte self-message.
    - pingpong_8B: Send/Recv_enqueue between 2 ranks sharing GPU 0 (half RTT).
    - allreduce_4KiB_P2: Allreduce_enqueue (fused single launch), 2 ranks.
    """
    import torch

    def world(P):
        w = mpix.World(P, [0] * P)
        ctx = {}

        def setup(r):
            s = mpix.testing.new_stream(0)
            ctx[r] = (s, w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s, mpix_graph="1")))
        w.run_ranks(setup)
        return w, ctx

    def timed(w, ctx, step, P):
        """step(r, k): enqueue k iterations on rank r's stream. Returns the max
        over ranks of the stream time for R*G iterations (seconds)."""
        ev = {r: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for r in range(P)}

        def run(r):
            s = ctx[r][0]
            ev[r][0].record(s)
            for _ in range(R):
                step(r, G)
            ev[r][1].record(s)
        w.run_ranks(lambda r: step(r, 4))  # warm-up
        for r in range(P):
            ctx[r][0].synchronize()
        w.run_ranks(run)
        for r in range(P):
            ctx[r][0].synchronize()
        return max(ev[r][0].elapsed_time(ev[r][1]) for r in range(P)) / 1e3

    def both(w, ctx, P, enqueue):
        """enqueue(r, k) enqueues k iterations; returns (eager_us, graph_us)."""
        t_eager = timed(w, ctx, enqueue, P)
        execs = {}

        def cap(r):
            s = ctx[r][0]
            s.synchronize()
            mpix.testing.graph_begin(s)
            try:
                enqueue(r, G)
            finally:
                execs[r] = mpix.testing.graph_end(s)
        w.run_ranks(cap)

        def replay(r, k):
            s = ctx[r][0]
            for _ in range(max(1, k // G)):
                mpix.testing.graph_launch(execs[r], s)
        t_graph = timed(w, ctx, replay, P)
        for e in execs.values():
            mpix.testing.graph_destroy(e)
        n = R * G
        return t_eager / n * 1e6, t_graph / n * 1e6

    out = {"iterations_per_graph": G, "replays": R}
    w, ctx = world(1)
    a = torch.zeros(8, dtype=torch.uint8, device=0)
    b = torch.zeros(8, dtype=torch.uint8, device=0)
    c0 = ctx[0][1]

    def loop(r, k):
        for _ in range(k):
            rq = [c0.isend_enqueue(a, 8, mpix.MPI_BYTE, 0, 1),
                  c0.irecv_enqueue(b, 8, mpix.MPI_BYTE, 0, 1)]
            mpix.waitall_enqueue(rq)
    e, g = both(w, ctx, 1, loop)
    out["loopback_8B"] = {"eager_us": e, "graph_us": g}

    # in-stream chain: producer kernel -> Send_enqueue -> Recv_enqueue ->
    # consumer kernel (8 B self-message, one stream)
    x = torch.zeros(2, dtype=torch.float32, device=0)
    y = torch.zeros(2, dtype=torch.float32, device=0)
    s0 = ctx[0][0]

    def chain(r, k):
        for _ in range(k):
            mpix.testing.fill_f32(x, 2, 1.0, s0)
            c0.send_enqueue(x, 2, mpix.MPI_FLOAT, 0, 3)
            c0.recv_enqueue(y, 2, mpix.MPI_FLOAT, 0, 3)
            mpix.testing.saxpy(2, 1.0, y, x, s0)
    e, g = both(w, ctx, 1, chain)
    out["self_chain_8B"] = {"eager_us": e, "graph_us": g,
                            "kernels": "producer + send + recv + consumer"}
    w.finalize()

    w, ctx = world(2)
    bufs = {r: (torch.zeros(8, dtype=torch.uint8, device=0),
                torch.zeros(8, dtype=torch.uint8, device=0)) for r in range(2)}

    def pp(r, k):
        c = ctx[r][1]
        sb, rb = bufs[r]
        for _ in range(k):
            if r == 0:
                c.send_enqueue(sb, 8, mpix.MPI_BYTE, 1, 2)
                c.recv_enqueue(rb, 8, mpix.MPI_BYTE, 1, 3)
            else:
                c.recv_enqueue(rb, 8, mpix.MPI_BYTE, 0, 2)
                c.send_enqueue(sb, 8, mpix.MPI_BYTE, 0, 3)
    e, g = both(w, ctx, 2, pp)
    out["pingpong_8B_half_rtt"] = {"eager_us": e / 2, "graph_us": g / 2}

    xs = {r: (torch.ones(1024, device=0), torch.zeros(1024, device=0)) for r in range(2)}

    def ar(r, k):
        c = ctx[r][1]
        x, y = xs[r]
        for _ in range(k):
            c.allreduce_enqueue(x, y, 1024, mpix.MPI_FLOAT)
    e, g = both(w, ctx, 2, ar)
    out["allreduce_4KiB_P2"] = {"eager_us": e, "graph_us": g}
    for r in range(2):
        ctx[r][0].synchronize()
    w.finalize()
    return out
