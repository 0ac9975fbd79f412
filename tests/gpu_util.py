"""Shared helpers for the GPU tests: a world of P ranks (all on cuda:0 unless
more GPUs are visible), one torch stream + MPIX GPU stream + stream
communicator per rank, built collectively with run_ranks like the
reference's tests build theirs (proj/tests/test_comm.cpp)."""
import contextlib

import torch

from paper_2208_13707_b200 import mpix


class RankCtx:
    def __init__(self, rank, device, stream, mstream, comm, world_comm):
        self.rank = rank
        self.device = device
        self.stream = stream          # torch.cuda.Stream
        self.mstream = mstream        # mpix.Stream
        self.comm = comm              # stream communicator (enqueue-capable)
        self.world_comm = world_comm


@contextlib.contextmanager
def gpu_world(P, devices=None, spread=False):
    ndev = torch.cuda.device_count()
    if devices is None:
        devices = [(r % ndev) if spread else 0 for r in range(P)]
    w = mpix.World(P, devices)
    ctxs = [None] * P
    try:
        def setup(r):
            dev = devices[r]
            with torch.cuda.device(dev):
                s = mpix.testing.new_stream(dev)
            ms = mpix.Stream.from_cuda(s)
            wc = w.comm(r)
            c = wc.stream_comm_create(ms)
            ctxs[r] = RankCtx(r, dev, s, ms, c, wc)

        w.run_ranks(setup)
        yield w, ctxs
        for c in ctxs:
            c.stream.synchronize()
        for d in set(devices):
            torch.cuda.synchronize(d)
        # no spinning kernel of this test gave up on its watchdog
        errs = [mpix.rank_error(r) for r in range(P)]
        assert not any(errs), f"device watchdog fired: rank error words {errs}"
    finally:
        for d in set(devices):
            torch.cuda.synchronize(d)
        w.finalize()


def sync_all(ctxs):
    for c in ctxs:
        c.stream.synchronize()
