"""Bounded model check of SPEC.md:437 ("No deadlock for well-paired programs:
any schedule in which every enqueue op has a peer eventually reaches full
completion (bounded model check over <=4-op programs, 2 ranks)").

A program: 2 ranks, each with 2 enqueue communicators (one MPIX stream
each, so one CUDA stream each); at most 4 point-to-point operations in
total, every send paired with a receive on the same communicator with the
same (source, destination, tag) — self-messages included. Each stream ends
with one Waitall_enqueue over its non-blocking requests.

The reference semantics used to decide which programs complete (the
reference's queue worker, proj/src/exec_queue.cpp:27-46, running
proj/src/proc_enqueue.cpp:30-141 items in FIFO order):
- Send_enqueue / Isend_enqueue / Irecv_enqueue: post at their queue position
  and let the queue go on (sends are eager, proc_p2p.cpp:60-62);
- Recv_enqueue blocks its queue until its matched send has been posted;
- Waitall_enqueue blocks until every receive it names is matched.
Matching of concrete patterns is non-overtaking per (comm, source, dest,
tag): the k-th receive takes the k-th send (endpoint.cpp:29-69; checked
against the reference matcher by tests/test_oracle.py). A program whose
simulation stalls (a blocking receive ahead of its own send on one queue,
Appendix A13) deadlocks in the reference too and is excluded.
"""
import itertools

KINDS = ("Send", "Isend", "Recv", "Irecv")


def pairs_2():
    """Every (comm, src, dst, tag, send_kind, recv_kind) message."""
    for comm, src, dst, tag in itertools.product((0, 1), (0, 1), (0, 1), (0, 1)):
        for sk, rk in itertools.product(("Send", "Isend"), ("Recv", "Irecv")):
            yield (comm, src, dst, tag, sk, rk)


def programs(max_msgs=2, tags=(0, 1)):
    """Yield programs as {(rank, comm): [op, ...]} with op = (kind, peer, tag,
    msg_id). Every ordering of each rank-stream's operations is produced
    (orderings across different streams do not change the program)."""
    msgs = [m for m in pairs_2() if m[3] in tags]
    seen = set()
    for k in range(1, max_msgs + 1):
        for combo in itertools.combinations_with_replacement(range(len(msgs)), k):
            ms = [msgs[i] for i in combo]
            ops = {}
            for j, (comm, src, dst, tag, sk, rk) in enumerate(ms):
                ops.setdefault((src, comm), []).append((sk, dst, tag, j))
                ops.setdefault((dst, comm), []).append((rk, src, tag, j))
            keys = sorted(ops)
            for perms in itertools.product(*[itertools.permutations(ops[q]) for q in keys]):
                prog = {q: list(p) for q, p in zip(keys, perms)}
                canon = tuple((q, tuple((o[0], o[1], o[2], ms[o[3]][4:]) for o in prog[q])) for q in keys)
                sig = (canon, tuple(sorted(ms)))
                if sig in seen:
                    continue
                seen.add(sig)
                yield prog, ms


def expected_pairs(prog):
    """Receive op -> matched send op, both as (rank, comm, position): the
    k-th receive of (comm, src, dst, tag) takes the k-th send."""
    sends, recvs = {}, {}
    for (rank, comm), ops in prog.items():
        for pos, (kind, peer, tag, _) in enumerate(ops):
            if kind in ("Send", "Isend"):
                sends.setdefault((comm, rank, peer, tag), []).append((rank, comm, pos))
            else:
                recvs.setdefault((comm, peer, rank, tag), []).append((rank, comm, pos))
    out = {}
    for key, rl in recvs.items():
        sl = sends.get(key, [])
        for i, r in enumerate(rl):
            out[r] = sl[i] if i < len(sl) else None
    return out


def completes(prog):
    """Simulate the reference queues (see module doc): True if every queue
    drains, including its closing Waitall."""
    match = expected_pairs(prog)
    if any(v is None for v in match.values()):
        return False
    posted = set()  # sends posted, as (rank, comm, pos)
    queues = {q: list(range(len(ops))) + ["W"] for q, ops in prog.items()}
    irecvs = {q: [(q[0], q[1], p) for p, o in enumerate(ops) if o[0] == "Irecv"] for q, ops in prog.items()}
    progress = True
    while progress:
        progress = False
        for q, items in queues.items():
            while items:
                head = items[0]
                if head == "W":
                    if all(match[r] in posted for r in irecvs[q]):
                        items.pop(0)
                        progress = True
                        continue
                    break
                kind = prog[q][head][0]
                me = (q[0], q[1], head)
                if kind in ("Send", "Isend"):
                    posted.add(me)
                elif kind == "Recv" and match[me] not in posted:
                    break
                items.pop(0)
                progress = True
    return all(not v for v in queues.values())
