"""GPU: BASELINE.json configs 4 and 5 end to end, checked against the oracle.

cfg5 (halo stencil): 8 ranks in a 2x2x2 periodic decomposition (all on the
visible GPUs). After every exchange each halo must equal the neighbour's
boundary layer bit for bit; the stencil is bit-exact with orc_stencil7 (no
FMA contraction on either side), so after k steps the whole distributed field
equals the oracle's global periodic stencil.
cfg4 (message rate): 8 ranks x 4 stream comms, ring neighbours, window 64;
every 8-byte payload must arrive.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2208_13707_b200 import mpix
from paper_2208_13707_b200.workloads import HaloStencil, coords, msgrate
from tests.gpu_util import gpu_world, sync_all

pytestmark = pytest.mark.gpu


def global_step(g, w0, w1):
    """Oracle: one periodic 7-point step of the global field g (N^3),
    through orc_stencil7 on a padded copy."""
    N = g.shape[0]
    p = np.pad(g, 1, mode="wrap").astype(np.float32)
    out = O.stencil7(p.reshape(-1), N, N, N, w0, w1).reshape(N + 2, N + 2, N + 2)
    return out[1:-1, 1:-1, 1:-1].copy()


@pytest.mark.parametrize("pipelined", [False, True], ids=["seq", "pipe"])
@pytest.mark.parametrize("native", [False, True], ids=["python", "native"])
@pytest.mark.parametrize("n", [2, 3, 6, 17, 40])
def test_halo_stencil_matches_global_oracle(n, native, pipelined):
    """native: the same steps through the C++ driver (MPIXT_Halo_steps).
    pipelined: interior [2, n-1]^3 on a second stream during the exchange,
    boundary shell after the unpack — must equal the sequential step bit for
    bit (n = 2, 3: empty / one-point interior)."""
    P = 8
    N = 2 * n
    rng = np.random.default_rng(n)
    g = rng.uniform(-1, 1, (N, N, N)).astype(np.float32)  # [z][y][x]
    with gpu_world(P) as (w, ctx):
        blocks = []
        for r in range(P):
            b = HaloStencil(r, n, ctx[r].stream, ctx[r].comm, pipelined=pipelined)
            cx, cy, cz = coords(r)
            pad = np.zeros((n + 2, n + 2, n + 2), dtype=np.float32)
            pad[1:-1, 1:-1, 1:-1] = g[cz * n:(cz + 1) * n, cy * n:(cy + 1) * n, cx * n:(cx + 1) * n]
            b.u.copy_(torch.from_numpy(pad.reshape(-1)).to(0))
            blocks.append(b)
        torch.cuda.synchronize()
        steps = 3
        if native:
            mpix.testing.halo_steps(blocks, steps, [0] * P,
                                    mpix.testing.HALO_PIPE if pipelined else mpix.testing.HALO_SEQ)
        else:
            w.run_ranks(lambda r: [blocks[r].step() for _ in range(steps)])
        sync_all(ctx)
        exp = g
        for _ in range(steps):
            exp = global_step(exp, HaloStencil.W0, HaloStencil.W1)
        got = np.zeros_like(g)
        for r in range(P):
            cx, cy, cz = coords(r)
            blk = blocks[r].u.cpu().numpy().reshape(n + 2, n + 2, n + 2)[1:-1, 1:-1, 1:-1]
            got[cz * n:(cz + 1) * n, cy * n:(cy + 1) * n, cx * n:(cx + 1) * n] = blk
        assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))


def test_halo_faces_bit_exact_after_exchange():
    P, n = 8, 9
    with gpu_world(P) as (w, ctx):
        blocks = [HaloStencil(r, n, ctx[r].stream, ctx[r].comm) for r in range(P)]
        for r, b in enumerate(blocks):
            b.u.copy_(torch.arange(b.u.numel(), dtype=torch.float32, device=0) + 1000 * r)
        torch.cuda.synchronize()
        w.run_ranks(lambda r: blocks[r].exchange())
        sync_all(ctx)
        from paper_2208_13707_b200.workloads import OPP, neighbour
        for r in range(P):
            for d in range(6):
                q = neighbour(r, d)
                # my halo d == neighbour's packed face OPP(d) (its interior layer)
                assert torch.equal(blocks[r].rbuf[d].cpu(), blocks[q].sbuf[OPP[d]].cpu()), (r, d)


def test_msgrate_ring_all_messages_arrive():
    P, S, W, B = 8, 4, 64, 3
    with gpu_world(P) as (w, ctx0):
        ctxs = [[] for _ in range(P)]
        bufs = [[] for _ in range(P)]

        def setup(r):
            for k in range(S):
                s = mpix.testing.new_stream(0)
                c = w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s))
                ctxs[r].append((s, c))

        # comm creation is collective per stream index: all ranks create comm k together
        w.run_ranks(setup)
        for r in range(P):
            for k in range(S):
                sb = torch.tensor([r, k], dtype=torch.int32, device=0)
                rb = torch.full((W, 2), -1, dtype=torch.int32, device=0)
                bufs[r].append((sb, rb))
        torch.cuda.synchronize()
        res = msgrate(w, ctxs, S, W, B, bufs)
        torch.cuda.synchronize()
        assert res["messages"] == P * S * W * B
        for r in range(P):
            left = (r + P - 1) % P
            for k in range(S):
                rb = bufs[r][k][1].cpu()
                assert bool((rb[:, 0] == left).all()) and bool((rb[:, 1] == k).all()), (r, k)


@pytest.mark.parametrize("n", [1, 2, 5, 33, 70])
def test_stencil_box_plus_shell_is_the_whole_update(n):
    """The interior box kernel and the shell kernel write disjoint points whose
    union is the block's interior: together they equal orc_stencil7 on the
    whole block, and the halo of out stays untouched."""
    rng = np.random.default_rng(n)
    N3 = (n + 2) ** 3
    u_h = rng.uniform(-1, 1, N3).astype(np.float32)
    exp = O.stencil7(u_h, n, n, n, HaloStencil.W0, HaloStencil.W1)
    u = torch.from_numpy(u_h).to(0)
    s = torch.cuda.current_stream()
    for how in ("full", "split"):
        out = torch.full((N3,), 7.0, dtype=torch.float32, device=0)
        if how == "full":
            mpix.testing.stencil7(u, out, n, n, n, HaloStencil.W0, HaloStencil.W1, s)
        else:
            mpix.testing.stencil7_box(u, out, n, n, n, (2, n - 1) * 3, HaloStencil.W0,
                                      HaloStencil.W1, s)
            mpix.testing.stencil7_shell(u, out, n, n, n, HaloStencil.W0, HaloStencil.W1, s)
        torch.cuda.synchronize()
        got = out.cpu().numpy().reshape(n + 2, n + 2, n + 2)
        want = exp.reshape(n + 2, n + 2, n + 2).copy()
        inner = (slice(1, -1),) * 3
        assert np.array_equal(got[inner].view(np.uint32), want[inner].view(np.uint32)), how
        halo = np.ones_like(got, dtype=bool)
        halo[inner] = False
        assert (got[halo] == 7.0).all(), how
