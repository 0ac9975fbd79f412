"""Worker for tests/test_gpu_mp.py: one rank per process (torchrun), the
multi-process world (symmetric heap + MPIX_World_init_mp). Exercises the
enqueue p2p, conventional p2p and collectives across processes and checks
every result exactly; prints "MP OK <rank>" on success."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2208_13707_b200 import mpix  # noqa: E402


def main():
    dist.init_process_group("gloo")
    w = mpix.MPWorld(heap_bytes=3 << 30)  # arena (1 GiB) + buffers
    r, n, dev = w.rank, w.n, w.device
    peer = 1 - r if n == 2 else (r + 1) % n
    left = (r + n - 1) % n
    s = mpix.testing.new_stream(dev)
    c = w.comm().stream_comm_create(mpix.Stream.from_cuda(s))
    g = torch.Generator().manual_seed(1234)
    # deterministic per-rank payloads known to every rank
    pay = {q: torch.randint(0, 256, (6 << 20,), dtype=torch.uint8, generator=g) for q in range(n)}
    src = w.alloc(6 << 20)
    dst = w.alloc(6 << 20)
    src.copy_(pay[r].to(dev))
    torch.cuda.synchronize(dev)
    # 1. ring exchange of several sizes: Isend to the right, Irecv from the left
    for nb in (0, 8, 4096, 70000, 1 << 20, 6 << 20):
        dst.zero_()
        torch.cuda.synchronize(dev)
        rr = c.irecv_enqueue(dst, nb, mpix.MPI_BYTE, left, 3)
        rs = c.isend_enqueue(src, nb, mpix.MPI_BYTE, (r + 1) % n, 3)
        mpix.waitall_enqueue([rr, rs])
        s.synchronize()
        assert torch.equal(dst[:nb].cpu(), pay[left][:nb]), ("ring", nb)
    # 2. blocking ping-pong between ranks 0 and 1 (eager and staged sends)
    if r < 2 and n >= 2:
        for nb in (16, 100000, 3 << 20):
            for it in range(3):
                if r == 0:
                    c.send_enqueue(src, nb, mpix.MPI_BYTE, 1, 10 + it)
                    c.recv_enqueue(dst, nb, mpix.MPI_BYTE, 1, 20 + it)
                else:
                    c.recv_enqueue(dst, nb, mpix.MPI_BYTE, 0, 10 + it)
                    c.send_enqueue(dst, nb, mpix.MPI_BYTE, 0, 20 + it)
            s.synchronize()
            if r == 0:
                assert torch.equal(dst[:nb].cpu(), pay[0][:nb]), ("pingpong", nb)
    # 2b. a blocking send larger than an arena slot (64 MiB) before its
    #     receive is posted: staged through a heap staging buffer
    big = 80 << 20
    ref = pay[0].repeat(big // (6 << 20) + 1)[:big]
    if r < 2:
        bs = w.alloc(big)
        br = w.alloc(big)
        bs.copy_(ref.to(dev))
        torch.cuda.synchronize(dev)
    dist.barrier()
    if r == 0:
        c.send_enqueue(bs, big, mpix.MPI_BYTE, 1, 30)
        s.synchronize()  # completes before the receive exists: staged
    dist.barrier()
    if r == 1:
        c.recv_enqueue(br, big, mpix.MPI_BYTE, 0, 30)
        s.synchronize()
        assert torch.equal(br.cpu(), ref), "staged send > 64 MiB"
    dist.barrier()
    # 3. allreduce (fp32, exactly representable inputs: any order is exact)
    cnt = (1 << 20) + 5
    x = w.alloc(cnt, torch.float32)
    y = w.alloc(cnt, torch.float32)
    vals = [(torch.arange(cnt, dtype=torch.float32) % 1000 - 500 + q) / 4 for q in range(n)]
    x.copy_(vals[r].to(dev))
    torch.cuda.synchronize(dev)
    c.allreduce_enqueue(x, y, cnt, mpix.MPI_FLOAT)
    s.synchronize()
    exp = vals[0].clone()
    for q in range(1, n):
        exp += vals[q]
    assert torch.equal(y.cpu(), exp), "allreduce"
    # small (fused single-launch) allreduce
    c.allreduce_enqueue(x, y, 100, mpix.MPI_FLOAT)
    s.synchronize()
    assert torch.equal(y[:100].cpu(), exp[:100]), "allreduce small"
    # 4. bcast from the last rank and allgather
    b = w.alloc(1 << 20)
    b.copy_(pay[r][: 1 << 20].to(dev))
    torch.cuda.synchronize(dev)
    c.bcast_enqueue(b, 1 << 20, mpix.MPI_BYTE, n - 1)
    s.synchronize()
    assert torch.equal(b.cpu(), pay[n - 1][: 1 << 20]), "bcast"
    ag = w.alloc(n * 4096)
    c.allgather_enqueue(src, ag, 4096, mpix.MPI_BYTE)
    s.synchronize()
    assert torch.equal(ag.cpu(), torch.cat([pay[q][:4096] for q in range(n)])), "allgather"
    # alltoall: block q of rank r's sendbuf -> block r of rank q's recvbuf
    blk = 70000
    at = w.alloc(n * blk)
    c.alltoall_enqueue(src, at, blk, mpix.MPI_BYTE)
    s.synchronize()
    assert torch.equal(at.cpu(), torch.cat([pay[q][r * blk:(r + 1) * blk] for q in range(n)])), "alltoall"
    # 5. conventional p2p on the world comm
    wc = w.comm()
    if r < 2 and n >= 2:
        t = w.alloc(5000)
        if r == 0:
            wc.send(src, 5000, mpix.MPI_BYTE, 1, 7)
        else:
            wc.recv(t, 5000, mpix.MPI_BYTE, 0, 7)
            assert torch.equal(t.cpu(), pay[0][:5000]), "conventional"
    # 6. a non-heap receive buffer is rejected in multi-process mode
    plain = torch.zeros(64, dtype=torch.uint8, device=dev)
    try:
        c.irecv_enqueue(plain, 64, mpix.MPI_BYTE, left, 99)
        raise AssertionError("non-heap receive buffer accepted")
    except mpix.MPIXError as e:
        assert e.name == "INVALID_ARG", e.name
    # 7. CUDA-Graph capture across processes: a graph-capturable comm, a
    #    captured ring exchange + allreduce, replayed with device-side checks
    if os.environ.get("MPIX_MATCHING") == "dynamic":  # graph capture needs static matching
        gc = None
    else:
        s2 = mpix.testing.new_stream(dev)
        gc = w.comm().stream_comm_create(mpix.Stream.from_cuda(s2, mpix_graph="1"))
    if gc is not None:
        graph_section(w, gc, s2, r, n, left, dev)
    assert mpix.rank_error(r) == 0
    c.free()
    w.finalize()
    os.write(1, f"MP OK {r}\n".encode())  # one write: lines of ranks do not interleave
    dist.destroy_process_group()


def graph_section(w, gc, s2, r, n, left, dev):
    m = 70000
    gx = w.alloc(m, torch.float32)
    gy = w.alloc(m, torch.float32)
    gz = w.alloc(m, torch.float32)
    it = torch.zeros(1, dtype=torch.int32, device=dev)
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    torch.cuda.synchronize(dev)
    dist.barrier()
    mpix.testing.graph_begin(s2)
    mpix.testing.iter_fill(gx, m, it, float(r + 1), 1.0, s2)
    rq = [gc.irecv_enqueue(gy, m, mpix.MPI_FLOAT, left, 4),
          gc.isend_enqueue(gx, m, mpix.MPI_FLOAT, (r + 1) % n, 4)]
    mpix.waitall_enqueue(rq)
    mpix.testing.iter_check(gy, m, it, float(left + 1), 1.0, bad, s2)
    gc.allreduce_enqueue(gx, gz, m, mpix.MPI_FLOAT)
    mpix.testing.iter_check(gz, m, it, n * (n + 1) / 2, float(n), bad, s2)
    mpix.testing.iter_bump(it, s2)
    gexec = mpix.testing.graph_end(s2)
    for _ in range(6):
        mpix.testing.graph_launch(gexec, s2)
    s2.synchronize()
    mpix.testing.graph_destroy(gexec)
    assert it.item() == 6 and bad.item() == 0, ("graph", it.item(), bad.item())
    gc.free()


if __name__ == "__main__":
    main()
