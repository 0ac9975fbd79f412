"""Applications written against the enqueue API, used by the tests and
bench.py (BASELINE.json configs 4 and 5):

- `HaloStencil`: 3-D 7-point stencil on a 2x2x2 periodic decomposition. Each
  step packs the 6 faces, exchanges them with Isend/Irecv_enqueue +
  Waitall_enqueue, unpacks into the halos and runs the stencil, all in the
  rank's CUDA stream (no host synchronisation between steps).
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

    def __init__(self, rank: int, n: int, stream, comm, device=0, torch=None):
        import torch as _t
        self.t = torch or _t
        self.rank, self.n, self.stream, self.comm = rank, n, stream, comm
        shape = ((n + 2) * (n + 2) * (n + 2),)
        self.u = self.t.zeros(shape, dtype=self.t.float32, device=device)
        self.v = self.t.zeros(shape, dtype=self.t.float32, device=device)
        self.sbuf = [self.t.zeros(n * n, dtype=self.t.float32, device=device) for _ in range(6)]
        self.rbuf = [self.t.zeros(n * n, dtype=self.t.float32, device=device) for _ in range(6)]

    def exchange(self):
        n, s = self.n, self.stream
        for d in range(6):
            mpix.testing.halo_pack(self.u, n, n, n, d, self.sbuf[d], s)
        reqs = []
        for d in range(6):  # halo d is filled by the neighbour across d, which sent its OPP(d) face
            reqs.append(self.comm.irecv_enqueue(self.rbuf[d], n * n, mpix.MPI_FLOAT,
                                                neighbour(self.rank, d), OPP[d]))
        for d in range(6):
            reqs.append(self.comm.isend_enqueue(self.sbuf[d], n * n, mpix.MPI_FLOAT,
                                                neighbour(self.rank, d), d))
        mpix.waitall_enqueue(reqs)
        for d in range(6):
            mpix.testing.halo_unpack(self.u, n, n, n, d, self.rbuf[d], s)

    def step(self):
        self.exchange()
        mpix.testing.stencil7(self.u, self.v, self.n, self.n, self.n, self.W0, self.W1, self.stream)
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
