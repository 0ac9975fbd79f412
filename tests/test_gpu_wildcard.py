"""GPU parity of wildcard receives under dynamic matching (MPIX_MATCHING=dynamic,
SURVEY.md Appendix A4, §8(f) item 1).

The reference matches with one posted-receive queue and one unexpected queue
per endpoint (proj/src/endpoint.cpp:29-69); its outcome depends on the
interleaving of operations across ranks. The device engine serialises every
matching step of a receiver under a lock, so its outcome must be the
reference's outcome for SOME interleaving consistent with each rank's program
order. Oracle: `orc_match_reference` (oracle/streamix_oracle.c, pinned to the
reference's own outcomes by tests/test_oracle.py) over all interleavings.
"""
import itertools
import random

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2208_13707_b200 import mpix
from tests.gpu_util import gpu_world, sync_all

pytestmark = pytest.mark.gpu

ANY = -1
NONE = np.uint64(0xFFFFFFFFFFFFFFFF)


@pytest.fixture(autouse=True)
def dynamic(monkeypatch):
    monkeypatch.setenv("MPIX_MATCHING", "dynamic")


def outcomes(progs):
    """Every outcome of the reference matcher over all interleavings."""
    base = [r for r, p in enumerate(progs) for _ in p]
    seen = set()
    for o in set(itertools.permutations(base)):
        pairs = O.match_reference(progs, list(o))
        seen.add(pairs.tobytes())
    return seen


def run_program(progs, nbytes=8, sizes=None):
    """Execute per-rank programs of (is_send, peer, tag) as Isend/Irecv_enqueue
    + one Waitall per rank; return the pairs matrix in the oracle's layout
    (receive -> send op id) from the delivered payloads."""
    P = len(progs)
    max_pos = max(1, max(len(p) for p in progs))
    with gpu_world(P) as (w, ctx):
        bufs = {}
        for r, prog in enumerate(progs):
            for i, (is_send, peer, tag) in enumerate(prog):
                n = sizes[(r, i)] if sizes else nbytes
                if is_send:
                    t = torch.full((n // 8,), (r << 16) | i, dtype=torch.int64, device=0)
                else:
                    t = torch.full((n // 8,), -1, dtype=torch.int64, device=0)
                bufs[(r, i)] = (t, n)
        torch.cuda.synchronize()

        def body(r):
            c = ctx[r].comm
            reqs = []
            for i, (is_send, peer, tag) in enumerate(progs[r]):
                t, n = bufs[(r, i)]
                if is_send:
                    reqs.append(c.isend_enqueue(t, n, mpix.MPI_BYTE, peer, tag))
                else:
                    reqs.append(c.irecv_enqueue(t, n, mpix.MPI_BYTE, peer, tag))
            mpix.waitall_enqueue(reqs)

        w.run_ranks(body)
        sync_all(ctx)
        for r in range(P):
            assert mpix.rank_error(r) == 0, r
        pairs = np.full((P, max_pos), NONE, dtype=np.uint64)
        for r, prog in enumerate(progs):
            for i, (is_send, _, _) in enumerate(prog):
                if not is_send:
                    t, n = bufs[(r, i)]
                    v = t.cpu().numpy()
                    sid = int(v[0])
                    assert sid >= 0, "receive not delivered"
                    slen = bufs[(sid >> 16, sid & 0xffff)][1]
                    k = min(slen, n) // 8  # truncation: endpoint.cpp:17-24
                    assert (v[:k] == sid).all() and (v[k:] == -1).all(), "torn payload"
                    pairs[r, i] = np.uint64(sid)
        return pairs


def complete(progs):
    """True if every receive is matched in every interleaving (no hang)."""
    for o in outcomes(progs):
        pairs = np.frombuffer(o, dtype=np.uint64).reshape(len(progs), -1)
        for r, prog in enumerate(progs):
            for i, (is_send, _, _) in enumerate(prog):
                if not is_send and pairs[r, i] == NONE:
                    return False
    return True


def test_any_tag_keeps_send_order():
    """Irecv(src, ANY_TAG) x4 take a source's messages in send order
    (non-overtaking, endpoint.cpp:46-69)."""
    progs = [[(1, 1, 5), (1, 1, 3), (1, 1, 5), (1, 1, 7)],
             [(0, 0, ANY), (0, 0, ANY), (0, 0, ANY), (0, 0, ANY)]]
    assert complete(progs)
    got = run_program(progs)
    assert got.tobytes() in outcomes(progs)
    assert [int(x) & 0xffff for x in got[1]] == [0, 1, 2, 3]


def test_concrete_receive_posted_before_wildcard_wins():
    """A receive for tag 3 posted before an ANY_TAG receive takes the tag-3
    message even though the tag-5 message was sent first."""
    progs = [[(1, 1, 5), (1, 1, 3)], [(0, 0, 3), (0, 0, ANY)]]
    got = run_program(progs)
    assert got.tobytes() in outcomes(progs)
    assert int(got[1, 0]) & 0xffff == 1 and int(got[1, 1]) & 0xffff == 0


def test_any_source_from_three_senders():
    progs = [[(0, ANY, 1), (0, ANY, 1), (0, ANY, ANY)], [(1, 0, 1)], [(1, 0, 1)], [(1, 0, 9)]]
    assert complete(progs)
    got = run_program(progs)
    assert got.tobytes() in outcomes(progs)


@pytest.mark.parametrize("seed", range(12))
def test_random_programs_match_reference(seed):
    """Random 2-3 rank programs mixing concrete and wildcard receives: the
    device outcome is one of the reference matcher's outcomes."""
    rng = random.Random(seed)
    for _ in range(200):
        P = rng.choice([2, 3])
        progs = [[] for _ in range(P)]
        nsend = rng.randint(1, 3)
        for _ in range(nsend):
            s = rng.randrange(P)
            d = rng.choice([q for q in range(P) if q != s] or [s])
            tag = rng.choice([0, 1])
            progs[s].append((1, d, tag))
            # the matching receive, possibly wildcarded
            src = rng.choice([s, ANY])
            tg = rng.choice([tag, ANY])
            progs[d].append((0, src, tg))
        for p in progs:
            rng.shuffle(p)
        if sum(len(p) for p in progs) <= 8 and complete(progs):
            break
    else:
        pytest.skip("no complete program drawn")
    got = run_program(progs)
    assert got.tobytes() in outcomes(progs), (progs, got)


@pytest.mark.parametrize("inline", ["65536", "0"])
def test_wildcards_with_large_and_truncated_messages(inline, monkeypatch):
    """Grouped copies and truncation with ANY_SOURCE / ANY_TAG receives."""
    monkeypatch.setenv("MPIX_INLINE_BYTES", inline)
    big = (2 << 20) + 8
    progs = [[(1, 2, 4), (1, 2, 4)], [(1, 2, 6)], [(0, ANY, ANY), (0, 0, ANY), (0, ANY, ANY)]]
    assert complete(progs)
    sizes = {(0, 0): big, (0, 1): 64, (1, 0): 4096, (2, 0): big, (2, 1): big, (2, 2): 4096}
    got = run_program(progs, sizes=sizes)
    assert got.tobytes() in outcomes(progs)


def test_blocking_wildcard_recv_and_staged_sends():
    """Blocking Recv_enqueue(ANY_SOURCE, ANY_TAG) against eager and staged
    blocking Send_enqueue from two ranks (dynamic staged publication)."""
    sizes = [16, 3 << 20]
    with gpu_world(3) as (w, ctx):
        src = {r: torch.full((sizes[r - 1] // 8,), r, dtype=torch.int64, device=0) for r in (1, 2)}
        dst = [torch.zeros((3 << 20) // 8, dtype=torch.int64, device=0) for _ in range(2)]
        torch.cuda.synchronize()

        def body(r):
            c = ctx[r].comm
            if r == 0:
                for k in range(2):
                    c.recv_enqueue(dst[k], 3 << 20, mpix.MPI_BYTE, mpix.MPI_ANY_SOURCE, mpix.MPI_ANY_TAG)
            else:
                c.send_enqueue(src[r], sizes[r - 1], mpix.MPI_BYTE, 0, 10 + r)

        w.run_ranks(body)
        sync_all(ctx)
        got = sorted(int(d[0]) for d in dst)
        assert got == [1, 2]
        for d in dst:
            r = int(d[0])
            n = sizes[r - 1] // 8
            assert bool((d[:n] == r).all())
        for r in range(3):
            assert mpix.rank_error(r) == 0


def test_static_mode_rejects_wildcards(monkeypatch):
    monkeypatch.setenv("MPIX_MATCHING", "static")
    with gpu_world(1) as (w, ctx):
        t = torch.zeros(8, dtype=torch.uint8, device=0)
        with pytest.raises(mpix.MPIXError):
            ctx[0].comm.irecv_enqueue(t, 8, mpix.MPI_BYTE, mpix.MPI_ANY_SOURCE, 0)


def test_stream_hint_selects_dynamic_matching(monkeypatch):
    """info "mpix_matching"="dynamic" on one member's stream makes the comm
    wildcard-capable for every member (agreed at MPIX_Stream_comm_create)."""
    monkeypatch.setenv("MPIX_MATCHING", "static")
    w = mpix.World(2, [0, 0])
    try:
        comms = {}

        def setup(r):
            s = mpix.testing.new_stream(0)
            hints = {"mpix_matching": "dynamic"} if r == 1 else {}
            comms[r] = (s, w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s, **hints)))

        w.run_ranks(setup)
        x = torch.full((4,), 7, dtype=torch.int64, device=0)
        y = torch.zeros(4, dtype=torch.int64, device=0)
        torch.cuda.synchronize()

        def body(r):
            s, c = comms[r]
            if r == 0:
                c.send_enqueue(x, 32, mpix.MPI_BYTE, 1, 3)
            else:
                c.recv_enqueue(y, 32, mpix.MPI_BYTE, mpix.MPI_ANY_SOURCE, mpix.MPI_ANY_TAG)

        w.run_ranks(body)
        for r in range(2):
            comms[r][0].synchronize()
        assert torch.equal(x.cpu(), y.cpu())
    finally:
        torch.cuda.synchronize()
        w.finalize()


def test_bad_matching_hint_is_bad_hint():
    info = mpix.cuda_stream_info(mpix.testing.new_stream(0))
    info.set("mpix_matching", "sometimes")
    with pytest.raises(mpix.MPIXError) as e:
        mpix.Stream(info)
    assert e.value.name == "BAD_HINT"
