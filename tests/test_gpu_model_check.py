"""GPU: bounded model check of SPEC.md:434-437 over every 2-rank program of
at most 4 point-to-point enqueue operations (tests/model_check.py): two
enqueue communicators (CUDA streams) per rank, Send/Isend/Recv/Irecv_enqueue
with concrete tags 0/1, self-messages included, a closing Waitall_enqueue per
stream. Every program the reference completes (its queue semantics,
proj/src/exec_queue.cpp:27-46 + proj/src/proc_enqueue.cpp:30-141) must
complete here under a short watchdog, and every receive must hold the
payload of the send the reference's non-overtaking matcher pairs it with
(proj/src/endpoint.cpp:29-69). Run with coalesced launches (default) and
with one launch per operation (MPIX_BATCH=0), at an eager size, a large
(copy-grid) size, and a staged size above the device arena slot.
"""
import contextlib
import os
import random

import pytest
import torch

from paper_2208_13707_b200 import mpix
from tests import model_check as M

pytestmark = pytest.mark.gpu

MAXPOS = 4


@contextlib.contextmanager
def env(**kv):
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update({k: str(v) for k, v in kv.items()})
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def run_all(progs, nbytes, batch):
    with env(MPIX_BATCH=batch, MPIX_SPIN_TIMEOUT_MS=5000):
        w = mpix.World(2, [0, 0])
    try:
        st, cm = {}, {}

        def setup(r):
            for c in range(2):
                s = mpix.testing.new_stream(0)
                st[(r, c)] = s
                cm[(r, c)] = w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s))

        w.run_ranks(setup)
        n = max(nbytes, 8)
        send = torch.empty((2, 2, MAXPOS, n), dtype=torch.uint8, device=0)
        for r, c, p in ((r, c, p) for r in range(2) for c in range(2) for p in range(MAXPOS)):
            mpix.testing.fill_pattern(send[r, c, p], n, 1000 + 100 * r + 10 * c + p, 0,
                                      torch.cuda.current_stream())
        recv = torch.zeros((2, 2, MAXPOS, n), dtype=torch.uint8, device=0)
        torch.cuda.synchronize()
        for k, (prog, _) in enumerate(progs):
            recv.zero_()
            torch.cuda.synchronize()
            for (r, c), ops in prog.items():
                comm = cm[(r, c)]
                reqs = []
                for pos, (kind, peer, tag, _) in enumerate(ops):
                    if kind == "Send":
                        comm.send_enqueue(send[r, c, pos], nbytes, mpix.MPI_BYTE, peer, tag)
                    elif kind == "Isend":
                        reqs.append(comm.isend_enqueue(send[r, c, pos], nbytes, mpix.MPI_BYTE, peer, tag))
                    elif kind == "Recv":
                        comm.recv_enqueue(recv[r, c, pos], nbytes, mpix.MPI_BYTE, peer, tag)
                    else:
                        reqs.append(comm.irecv_enqueue(recv[r, c, pos], nbytes, mpix.MPI_BYTE, peer, tag))
                if reqs:
                    mpix.waitall_enqueue(reqs)
            for s in st.values():
                s.synchronize()
            for q in cm.values():
                q.check()  # no watchdog fired: the program completed
            for (rr, rc, rp), snd in M.expected_pairs(prog).items():
                sr, sc, sp = snd
                assert torch.equal(recv[rr, rc, rp, :nbytes], send[sr, sc, sp, :nbytes]), \
                    (k, prog, (rr, rc, rp), snd)
    finally:
        torch.cuda.synchronize()
        w.finalize()


def completing(max_msgs=2):
    return [(p, m) for p, m in M.programs(max_msgs) if M.completes(p)]


@pytest.mark.parametrize("batch", [1, 0], ids=["coalesced", "per-op"])
@pytest.mark.parametrize("nbytes", [8, 256 << 10], ids=["eager", "large"])
def test_every_completing_program_completes_with_the_reference_matching(nbytes, batch):
    progs = completing()
    assert len(progs) == 6864
    run_all(progs, nbytes, batch)


@pytest.mark.parametrize("batch", [1, 0], ids=["coalesced", "per-op"])
def test_staged_sizes_sample(batch):
    """6 MiB blocking sends exceed the 4 MiB arena slot (host staging
    buffers); a seeded sample of the same programs."""
    progs = completing()
    random.Random(5).shuffle(progs)
    run_all(progs[:400], 6 << 20, batch)
