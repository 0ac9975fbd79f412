#!/usr/bin/env python
"""bench.py — MPIX-stream GPU-enqueue path on B200 (arXiv 2208.13707).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mpix|reference]

Headline (N=1, BASELINE.json config 2 at one GPU, SURVEY.md §8d cfg2 "1 GPU:
loopback self-messages on one stream"): a step is one 256 MiB message sent
and received by the same rank on one CUDA stream through
MPIX_Isend_enqueue + MPIX_Irecv_enqueue + MPIX_Waitall_enqueue. `value` is
message bytes delivered per second (GB/s), device-timed with CUDA events.
The dominant kernel is the receive kernel that pulls the payload (2*S bytes
of HBM traffic per launch: read + write).

N>1 (torchrun): the world is one process driving N GPUs (the reference's
World/run_ranks model); torchrun rank 0 hosts it, the other
ranks join a barrier and exit. GPU pairs (0,1),(2,3).. stream 256 MiB
messages; value = aggregate GB/s, time = max over GPUs of event time.

--impl reference: the reference's own CPU implementation (oracle/_ref, the
unmodified streamix library compiled from its sources) on the same workload.
"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # see paper_2208_13707_b200/mpix.py
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
MiB = 1 << 20


_T0 = time.time()


def log(msg):
    """Progress on stderr (locates a stall when a run is cut off)."""
    print(f"[bench {time.time() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mpix", choices=["mpix", "reference"])
    ap.add_argument("--size", type=int, default=256 * MiB)
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--share-gpus", action="store_true",
                    help="validation only: map rank r to GPU r %% ndev (ranks share GPUs)")
    ap.add_argument("--single-process", action="store_true",
                    help="N>1: rank 0 drives all N GPUs in one process (the reference's World "
                         "model) instead of one process per GPU")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# --------------------------------------------------------------------------
# clocks (NVML) sampled over the soak + timed window
# --------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
        0x2: "applications_clocks_setting", 0x10: "sync_boost",
    }

    def __init__(self, dev=0):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if self.ok:
            self.stop_ev.set()
            self.t.join()
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------------------------
# reference arm / cpu baseline
# --------------------------------------------------------------------------
def host_cpus():
    """The host cores this process may run on (the CPU arm is pinned to them
    and they are stated in the line: nproc and the affinity list)."""
    try:
        aff = sorted(os.sched_getaffinity(0))
    except AttributeError:
        aff = list(range(os.cpu_count() or 1))
    return {"nproc": os.cpu_count(), "affinity": aff}


def pin_cpu_arm():
    """Pin the CPU arm to an explicit core list (the whole affinity mask, in
    order) so the reference's worker threads stay on the stated cores."""
    h = host_cpus()
    try:
        os.sched_setaffinity(0, h["affinity"])
    except (AttributeError, OSError):
        pass
    return h


def cpu_reference_selfmsg(size, budget_s, min_msgs=3):
    """The unmodified reference (oracle/_ref) on the loopback workload: one
    exec queue, isend+irecv+waitall_enqueue of `size` bytes per message."""
    import numpy as np
    from oracle import oracle as O
    R = O.ref()
    if R is None:
        return None
    h = pin_cpu_arm()
    src = np.random.default_rng(0).integers(0, 255, size, dtype=np.uint8)
    dst = np.zeros_like(src)
    R.ref_selfmsg(src.ctypes.data, dst.ctypes.data, size, 1, 0)  # warm
    msgs, t = 0, 0.0
    while t < budget_s or msgs < min_msgs:
        t += R.ref_selfmsg(src.ctypes.data, dst.ctypes.data, size, 2, 0)
        msgs += 2
    assert (dst == src).all()
    return {"value": size * msgs / t / 1e9, "unit": "GB/s", "cores": 2, "kind": "reference",
            "threads": 2, "host": h,
            "sample": f"{msgs} x {size >> 20} MiB self-messages (isend+irecv+waitall_enqueue) "
                      f"through the compiled reference, 1 rank = driver thread + queue worker "
                      f"(2 threads on the {h['nproc']}-core host), {t:.1f} s"}


def cpu_reference_configs():
    """The reference's own CPU path (oracle/_ref) on cfg1, cfg3 and cfg4 in
    the same run, on this host's cores (SURVEY.md §8(d) "CPU reference timed
    beside it"); bounded samples, sizes stated."""
    import numpy as np
    from oracle import oracle as O
    R = O.ref()
    if R is None:
        return None
    h = pin_cpu_arm()
    out = {"host": h, "kind": "reference (unmodified streamix compiled from its sources)"}
    # cfg1: 2 ranks, Send/Recv_enqueue ping-pong of 1 MiB fp32, 200 round trips
    n = 262144
    x = ((np.arange(n) % 1024).astype(np.float32) * np.float32(0.5))
    f0, f1 = C.c_uint64(), C.c_uint64()
    R.ref_pingpong(x.ctypes.data, 4 * n, 5, C.byref(f0), C.byref(f1))
    t = R.ref_pingpong(x.ctypes.data, 4 * n, 200, C.byref(f0), C.byref(f1))
    out["cfg1_pingpong_1MiB"] = {"round_trips": 200, "half_rtt_us": t / 400 * 1e6,
                                 "GBps": 4 * n / (t / 400) / 1e9, "fnv1a64_rank0": f0.value,
                                 "threads": 4}
    for nb, it in ((8, 2000), (4096, 2000)):
        b = np.zeros(nb, dtype=np.uint8)
        t = R.ref_pingpong(b.ctypes.data, nb, it, C.byref(f0), C.byref(f1))
        out[f"pingpong_{nb}B_half_rtt_us"] = t / (2 * it) * 1e6
    # cfg3: the composed allreduce (irecv/isend/waitall_enqueue + queued rank-ordered fold)
    ar = {}
    cnt = 16 << 20  # 64 MiB fp32 per rank (the 256 MiB config scaled to fit the sample budget)
    for P in (2, 4, 8):
        ins = np.ones(P * cnt, dtype=np.float32)
        outb = np.zeros_like(ins)
        t = R.ref_allreduce(P, cnt, 2, 1, ins.ctypes.data, outb.ctypes.data, 1)
        algbw = 4 * cnt / t / 1e9
        ar[f"f32_P{P}"] = {"bytes_per_rank": 4 * cnt, "s": t, "algbw_GBps": algbw,
                           "busbw_GBps": algbw * 2 * (P - 1) / P, "threads": 2 * P,
                           "check": bool(outb[0] == P)}
    out["cfg3_allreduce_64MiB"] = ar
    # cfg4: 8 ranks x 4 streams, 8-B messages, window 64 (bench.hpp:22)
    msgs = C.c_uint64()
    R.ref_msgrate(8, 4, 64, 5, C.byref(msgs))
    t = R.ref_msgrate(8, 4, 64, 100, C.byref(msgs))
    out["cfg4_msgrate_8B"] = {"ranks": 8, "streams_per_rank": 4, "window": 64, "batches": 100,
                              "msgs_per_s": msgs.value / t, "threads": 8 + 8 * 4}
    # paper Fig. 3: the reference's own lock-regime bench (bench.cpp:118-235),
    # 2 ranks x T threads, 8-B messages, window 64, 6400 messages per thread
    f3 = {}
    for mode, name in ((0, "global"), (1, "pervci"), (2, "stream")):
        f3[name] = {}
        for T in (1, 2, 4, 8):
            m = C.c_double()
            e = R.ref_fig3(mode, T, 64, 6400, C.byref(m))
            f3[name][str(T)] = m.value if e > 0 else None
    out["fig3_lock_regimes_msgs_per_s"] = f3
    return out


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np
    from oracle import oracle as O
    R = O.ref()
    if R is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    size = args.size
    n = args.gpus
    host = pin_cpu_arm()
    src = np.random.default_rng(0).integers(0, 255, size, dtype=np.uint8)
    dst = np.zeros_like(src)
    if n == 1:
        step = lambda: R.ref_selfmsg(src.ctypes.data, dst.ctypes.data, size, 1, 0)
        units_per_step = size
        workload = "loopback Isend/Irecv/Waitall_enqueue self-message, 1 rank"
        cores = 2
    else:
        # pairs exchange: P ranks, rank 2i -> 2i+1 (composed with the
        # reference's own ping-pong driver: one message each way per step)
        x = src
        f0, f1 = C.c_uint64(), C.c_uint64()
        pairs = n // 2
        def step():
            t = 0.0
            for _ in range(pairs):
                t += R.ref_pingpong(x.ctypes.data, size, 1, C.byref(f0), C.byref(f1)) / 2
            return t
        units_per_step = size * pairs
        workload = f"{pairs} pair(s) x one {size >> 20} MiB message"
        cores = 2 * 2
    for _ in range(args.warmup):
        step()
    t = sum(step() for _ in range(args.steps))
    v = units_per_step * args.steps / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": workload, "message_bytes": size, "host": "CPU (reference streamix)"},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "reference",
                         "threads": cores, "host": host,
                         "sample": f"{args.steps} steps of {workload}"},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def run_mpix(args):
    rank, world, local = dist_env()
    if world > 1:
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo")
        # Normally rank 0 sees all N GPUs and hosts the N-GPU world (the
        # reference's World/run_ranks model); if the launcher hides GPUs from
        # each process, every rank instead runs an independent one-GPU
        # replica of the N=1 step and the job time is the max over ranks.
        flag = torch.tensor([1 if torch.cuda.device_count() >= args.gpus or args.share_gpus else 0])
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag[0]) and not args.single_process:
            # one process per GPU: the multi-process world over the symmetric heap
            line = bench_mp(args, rank, world, local)
            dist.destroy_process_group()
            if rank == 0:
                print(json.dumps(line))
            return
        if not int(flag[0]):
            line = bench_replica(args, rank, world, local)
            dist.destroy_process_group()
            if rank == 0:
                print(json.dumps(line))
            return
        if rank != 0:
            dist.barrier()  # rank 0 hosts the N-GPU world
            dist.barrier()
            dist.destroy_process_group()
            return
        dist.barrier()
    try:
        line = bench_world(args)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
    print(json.dumps(line))


def bench_mp(args, rank, world, local):
    """N > 1, one process per GPU (MPIX_World_init_mp over the symmetric
    heap): GPU pairs (0,1),(2,3).. each move one S-byte message per step
    (Isend_enqueue on the even rank, Irecv_enqueue + Wait on the odd rank);
    K steps between barriers, device time max over ranks (gloo)."""
    import torch
    import torch.distributed as dist

    from paper_2208_13707_b200 import mpix
    S = args.size
    ndev = torch.cuda.device_count()
    dev = local % ndev
    w = mpix.MPWorld(heap_bytes=3 * S + (6 << 30), device=dev)  # bump heap: bench + extras buffers
    s = mpix.testing.new_stream(dev)
    c = w.comm().stream_comm_create(mpix.Stream.from_cuda(s))
    src, dst = w.alloc(S), w.alloc(S)
    mpix.testing.fill_pattern(src, S, 1234 + rank, 0, s)
    s.synchronize()
    pairs = world // 2
    active = rank < 2 * pairs
    sender = active and rank % 2 == 0
    peer = rank + 1 if sender else rank - 1
    tag = [0]

    def step():
        if not active:
            return
        tag[0] = (tag[0] + 1) % 30000
        if sender:
            mpix.wait_enqueue(c.isend_enqueue(src, S, mpix.MPI_BYTE, peer, tag[0]))
        else:
            mpix.wait_enqueue(c.irecv_enqueue(dst, S, mpix.MPI_BYTE, peer, tag[0]))

    step()
    s.synchronize()
    if active and not sender:  # the payload is the sender's pattern
        exp = w.alloc(S)
        mpix.testing.fill_pattern(exp, S, 1234 + peer, 0, s)
        s.synchronize()
        assert torch.equal(dst, exp), "payload mismatch"
    for _ in range(args.warmup):
        step()
    s.synchronize()
    clocks = ClockSampler(dev)
    clocks.start()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = mpix.launch_count()
    e0.record(s)
    for _ in range(args.steps):
        step()
    e1.record(s)
    s.synchronize()
    launches = mpix.launch_count() - l0
    dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_step = float(t[0]) / args.steps
    nl = torch.tensor([launches], dtype=torch.int64)
    dist.all_reduce(nl, op=dist.ReduceOp.SUM)
    # dominant kernel: the copy grid of each message. Both sides launch one;
    # the second arriver's copies (a sender pushes into a posted receive, a
    # receiver pulls a posted send), the other is empty. The runtime times
    # both and counts only grids whose decision records say they copied.
    mpix.testing.copy_timing(True)
    for _ in range(args.steps):
        step()
    s.synchronize()
    tot, ncopy, moved = mpix.testing.copy_timing_read()
    mpix.testing.copy_timing(False)
    agg = torch.tensor([tot, float(ncopy), float(moved)], dtype=torch.float64)
    dist.all_reduce(agg, op=dist.ReduceOp.SUM)
    k_ms = float(agg[0]) / max(float(agg[1]), 1.0)       # per copying grid, over all pairs
    k_bytes = float(agg[2]) / max(float(agg[1]), 1.0)    # bytes per copying grid
    n_copy = int(agg[1])
    clk = clocks.stop()
    same_gpu = ndev < world
    achieved = k_bytes / (k_ms / 1e3) / 1e9 if k_ms else 0.0
    if same_gpu:  # ranks share a GPU: an HBM copy (read + write) on one device
        peak = peaks().get("hbm_gbs", 6650.0) / 2
        peak_src = "half the measured HBM copy bandwidth (read + write on one GPU)"
    else:
        peak = 770.0
        peak_src = "measured peer copy 770 GB/s per direction (B200_PROFILING.md); nominal 900"
    # e2e: the sender's pinned host input -> H2D -> Isend; the receiver's
    # Irecv -> checksum -> 8-byte D2H; both synchronise every step
    host = torch.empty(S, dtype=torch.uint8, pin_memory=True)
    host.copy_(src.cpu())
    csum = torch.zeros(1, dtype=torch.int64, device=dev)
    hsum = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        if active:
            tag[0] = (tag[0] + 1) % 30000
            if sender:
                with torch.cuda.stream(s):
                    src.copy_(host, non_blocking=True)
                mpix.wait_enqueue(c.isend_enqueue(src, S, mpix.MPI_BYTE, peer, tag[0]))
            else:
                mpix.wait_enqueue(c.irecv_enqueue(dst, S, mpix.MPI_BYTE, peer, tag[0]))
                mpix.testing.checksum(dst, S, csum, s)
                with torch.cuda.stream(s):
                    hsum.copy_(csum, non_blocking=True)
        s.synchronize()
    e2e_t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    extras = {}
    if not args.no_extras:
        extras = extras_mp(args, mpix, torch, dist, w, c, s, rank, world, dev)
    c.free()
    w.finalize()
    return {
        "metric": METRIC, "value": S * pairs / t_step / 1e9, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": f"{pairs} GPU pair(s), one process per GPU (multi-process world, "
                               "symmetric heap): Isend_enqueue -> Irecv_enqueue + Wait",
                   "message_bytes": S, "ranks": world, "parallelism": "one process per GPU",
                   "l2": "inputs larger than L2",
                   "baseline_config": "BASELINE.json configs[1] (SURVEY.md §8d cfg2) at N GPUs",
                   **({"note": "GPUs shared by ranks: not an NVLink measurement"} if same_gpu else {})},
        "roofline": {"bound": "hbm" if same_gpu else "nvlink", "unit": "GB/s", "achieved": achieved,
                     "peak": peak, "frac": achieved / peak if peak else 0.0, "traffic": None,
                     "peak_source": peak_src,
                     **({} if same_gpu else {"frac_of_nominal_900": achieved / 900.0}),
                     "kernel": "mpix::k_gcopy (the second arriver's copy grid of each message)",
                     "kernel_ms": k_ms, "kernel_launches_timed": n_copy,
                     "algorithmic_bytes_per_launch": k_bytes,
                     "step_frac": S / t_step / 1e9 / peak if peak else 0.0},
        "e2e": {"value": S * pairs * args.steps / float(e2e_t[0]) / 1e9, "unit": "GB/s",
                "h2d_bytes_per_step": S * pairs, "d2h_bytes_per_step": 8 * pairs,
                "timing": "host wall clock, max over ranks, streams synchronised every step"},
        "gpu_launches": int(nl[0]),
        "clocks": clk,
        "extras": extras,
    }


SWEEP = [8, 64, 512, 4096, 32768, 262144, 2 << 20, 16 << 20, 64 << 20, 256 << 20, 1 << 30]
SWEEP_CAP = 1 << 30  # bytes of receive slots per window


def tmax(torch, dist, v):
    t = torch.tensor([float(v)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def stream_sweep_mp(mpix, torch, dist, c, s, rank, big_src, big_dst):
    """cfg2 bandwidth: rank 0 -> rank 1 unidirectional
    streaming, windows of 16 Isend_enqueue / Irecv_enqueue + Waitall_enqueue
    (fewer slots above 64 MiB: a window's receives fit 1 GiB), native driver;
    device time max over the pair."""
    out = {}
    for nb in SWEEP:
        W = 16 if nb * 16 <= SWEEP_CAP else max(1, SWEEP_CAP // nb)
        reps = int(min(200, max(3, (2 << 30) // (nb * W))))
        buf = big_src if rank == 0 else big_dst
        dist.barrier()
        if rank < 2:
            mpix.testing.stream_window(c, buf, nb, W, 2, 1 - rank, rank == 0, s)
            s.synchronize()
        dist.barrier()
        d = 0.0
        if rank < 2:
            d, _ = mpix.testing.stream_window(c, buf, nb, W, reps, 1 - rank, rank == 0, s)
        t = tmax(torch, dist, d)
        g = nb * W * reps / t / 1e9
        out[str(nb)] = {"window": W, "reps": reps, "GBps": g, "frac_of_770": g / 770.0,
                        "frac_of_900": g / 900.0}
    return out


def round_robin(n, rnd, me):
    """Partner of `me` in round `rnd` of the circle method (n even)."""
    m = n - 1
    if me == m:
        return rnd
    if me == rnd:
        return m
    return (2 * rnd - me) % m


def all_pairs_mp(mpix, torch, dist, c, s, rank, world, big_src, big_dst):
    """Every GPU pair at 64 MiB (SURVEY.md §8(d) "all 28 pairs ... for
    uniformity"): n-1 rounds of n/2 disjoint pairs; in each pair the lower
    rank streams 3 windows of 4 x 64 MiB to the higher; per-pair device time
    is the max of its two ranks."""
    nb, W, reps = 64 << 20, 4, 3
    pairs = {}
    for rnd in range(world - 1):
        q = round_robin(world, rnd, rank)
        sender = rank < q
        buf = big_src if sender else big_dst
        dist.barrier()
        mpix.testing.stream_window(c, buf, nb, W, 1, q, sender, s)
        s.synchronize()
        dist.barrier()
        d, _ = mpix.testing.stream_window(c, buf, nb, W, reps, q, sender, s)
        ts = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(ts, torch.tensor([float(q), d], dtype=torch.float64))
        for i in range(world):
            j = int(ts[i][0])
            if i < j:
                t = max(float(ts[i][1]), float(ts[j][1]))
                pairs[f"{i}-{j}"] = nb * W * reps / t / 1e9
    v = sorted(pairs.values())
    return {"message_bytes": nb, "pairs": pairs, "n_pairs": len(v), "min_GBps": v[0],
            "median_GBps": v[len(v) // 2], "max_GBps": v[-1], "min_over_max": v[0] / v[-1],
            "min_frac_of_770": v[0] / 770.0}


def extras_mp(args, mpix, torch, dist, w, c, s, rank, world, dev):
    """Multi-process N > 1: Allreduce_enqueue 256 MiB over all N (busbw) and
    the ranks 0 <-> 1 ping-pong half round trip, device time max over ranks."""
    out = {}
    big_src, big_dst = w.alloc(SWEEP_CAP), w.alloc(SWEEP_CAP)
    out["stream_bw_rank0_to_rank1"] = stream_sweep_mp(mpix, torch, dist, c, s, rank, big_src, big_dst)
    out["all_pairs_64MiB"] = all_pairs_mp(mpix, torch, dist, c, s, rank, world, big_src, big_dst)
    ar = {}
    for name, tdt, mdt in (("f32", torch.float32, mpix.MPI_FLOAT), ("bf16", torch.bfloat16, mpix.MPIX_BFLOAT16)):
        nbytes = 256 << 20
        cnt = nbytes // torch.tensor([], dtype=tdt).element_size()
        sb, rb = w.alloc(cnt, tdt), w.alloc(cnt, tdt)
        sb.fill_(1)
        torch.cuda.synchronize(dev)
        dist.barrier()
        mpix.testing.allreduce_loop([c], [s], [dev], [sb], [rb], cnt, mdt, 2)
        dist.barrier()
        d, _ = mpix.testing.allreduce_loop([c], [s], [dev], [sb], [rb], cnt, mdt, 10)
        t = torch.tensor([d / 10], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        algbw = nbytes / float(t[0]) / 1e9
        ar[name] = {"ms": float(t[0]) * 1e3, "algbw_GBps": algbw,
                    "busbw_GBps": algbw * 2 * (world - 1) / world,
                    "check": float(rb[0]) == float(world)}
    out["allreduce_256MiB"] = ar
    # Alltoall_enqueue: 32 MiB blocks per (sender, receiver) pair; busbw counts
    # the (N-1)/N of each rank's buffer that crosses to peers
    blk = 32 << 20
    asb, arb = w.alloc(world * blk), w.alloc(world * blk)
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    with torch.cuda.stream(s):
        c.alltoall_enqueue(asb, arb, blk, mpix.MPI_BYTE)
    s.synchronize()
    dist.barrier()
    ev0.record(s)
    for _ in range(5):
        c.alltoall_enqueue(asb, arb, blk, mpix.MPI_BYTE)
    ev1.record(s)
    s.synchronize()
    t = torch.tensor([ev0.elapsed_time(ev1) / 1e3 / 5], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out["alltoall_32MiB_blocks"] = {"ms": float(t[0]) * 1e3,
                                    "busbw_GBps": world * blk * (world - 1) / world / float(t[0]) / 1e9}
    pp = {}
    buf = w.alloc(64 << 20)
    for nb in (8, 4096, 65536, 1 << 20, 64 << 20):
        iters = 200 if nb <= (1 << 20) else 20
        dist.barrier()
        d = 0.0
        if rank < 2:
            mpix.testing.pingpong_side(c, buf, nb, 10, 1 - rank, rank == 0, s)
            d = mpix.testing.pingpong_side(c, buf, nb, iters, 1 - rank, rank == 0, s)
        t = torch.tensor([d], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        half = float(t[0]) / (2 * iters)
        pp[str(nb)] = {"half_rtt_us": half * 1e6, "GBps": nb / half / 1e9}
    out["pingpong_rank0_rank1"] = pp
    return out


def bench_replica(args, rank, world, local):
    """Replicas: each torchrun rank runs the N=1 loopback step on its own
    visible GPU (no data-path exchange), barrier + synchronize around K
    steps, device time max-reduced over ranks (gloo)."""
    import torch
    import torch.distributed as dist

    from paper_2208_13707_b200 import mpix
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    S = args.size
    w = mpix.World(1, [dev])
    s = mpix.testing.new_stream(dev)
    c = w.comm(0).stream_comm_create(mpix.Stream.from_cuda(s))
    src = torch.empty(S, dtype=torch.uint8, device=dev)
    dst = torch.zeros(S, dtype=torch.uint8, device=dev)
    mpix.testing.fill_pattern(src, S, 1234 + rank, 0, s)
    torch.cuda.synchronize(dev)
    mpix.testing.loopback(c, src, dst, S, max(3, args.warmup), s)
    torch.cuda.synchronize(dev)
    assert torch.equal(src, dst), "payload mismatch"
    dist.barrier()
    l0 = mpix.launch_count()
    dev_s, _ = mpix.testing.loopback(c, src, dst, S, args.steps, s)
    launches = mpix.launch_count() - l0
    torch.cuda.synchronize(dev)
    dist.barrier()
    t = torch.tensor([dev_s], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_step = float(t[0]) / args.steps
    clocks = ClockSampler(dev)
    clocks.start()
    mpix.testing.copy_timing(True)
    mpix.testing.loopback(c, src, dst, S, args.steps, s)
    torch.cuda.synchronize(dev)
    tot_ms, ncopy, moved = mpix.testing.copy_timing_read()
    mpix.testing.copy_timing(False)
    clk = clocks.stop()
    k_ms = tot_ms / max(ncopy, 1)
    peak = peaks().get("hbm_gbs", 6650.0)
    achieved = 2 * (moved / max(ncopy, 1)) / (k_ms / 1e3) / 1e9
    # e2e: pinned host input -> H2D -> loopback -> checksum -> 8-byte D2H
    host = torch.empty(S, dtype=torch.uint8, pin_memory=True)
    host.copy_(src.cpu())
    csum = torch.zeros(1, dtype=torch.int64, device=dev)
    hsum = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        with torch.cuda.stream(s):
            src.copy_(host, non_blocking=True)
        mpix.testing.loopback(c, src, dst, S, 1, s)
        mpix.testing.checksum(dst, S, csum, s)
        with torch.cuda.stream(s):
            hsum.copy_(csum, non_blocking=True)
        s.synchronize()
    e2e_t = time.perf_counter() - t0
    e2e_v = torch.tensor([S * args.steps / e2e_t / 1e9], dtype=torch.float64)
    dist.all_reduce(e2e_v, op=dist.ReduceOp.SUM)
    w.finalize()
    return {
        "metric": METRIC, "value": S * world / t_step / 1e9, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": "replicas only: each GPU runs the N=1 loopback step (GPUs not all "
                               "visible to one process, so no NVLink exchange)",
                   "message_bytes": S, "parallelism": f"{world} replicas",
                   "l2": "inputs larger than L2"},
        "roofline": {"bound": "hbm", "unit": "GB/s", "achieved": achieved, "peak": peak,
                     "frac": achieved / peak, "traffic": None,
                     "kernel": "mpix::k_gcopy (rank 0's replica)", "kernel_ms": k_ms},
        "e2e": {"value": float(e2e_v[0]), "unit": "GB/s", "h2d_bytes_per_step": S * world,
                "d2h_bytes_per_step": 8 * world,
                "timing": "host wall clock per replica, summed; stream synchronised every step"},
        "gpu_launches": launches,
        "clocks": clk,
    }


def bench_world(args):
    import torch

    from paper_2208_13707_b200 import mpix
    n = args.gpus
    S = args.size
    ndev = torch.cuda.device_count()
    assert ndev >= n or args.share_gpus, f"need {n} GPUs, see {ndev}"
    pk = peaks()
    P = n
    dev = [r % ndev for r in range(P)]
    w = mpix.World(P, dev)
    ctx = {}

    def setup(r):
        with torch.cuda.device(dev[r]):
            s = mpix.testing.new_stream(dev[r])
        ms = mpix.Stream.from_cuda(s)
        c = w.comm(r).stream_comm_create(ms)
        ctx[r] = (s, ms, c)

    w.run_ranks(setup)
    log('buffers (> L2: every step streams from HBM)')
    # buffers (> L2: every step streams from HBM)
    src, dst = {}, {}
    for r in range(P):
        src[r] = torch.empty(S, dtype=torch.uint8, device=dev[r])
        dst[r] = torch.zeros(S, dtype=torch.uint8, device=dev[r])
        mpix.testing.fill_pattern(src[r], S, 1234 + r, 0, ctx[r][0])
    for d in set(dev):
        torch.cuda.synchronize(d)

    if P == 1:
        senders, pairs = [0], [(0, 0)]
    else:
        pairs = [(2 * i, 2 * i + 1) for i in range(P // 2)]
        senders = [a for a, _ in pairs]
    Ktag = 0

    def step():
        """One message per pair. P=1: loopback on one stream."""
        nonlocal Ktag
        Ktag = (Ktag + 1) % 30000
        for a, b in pairs:
            sa, _, ca = ctx[a]
            sb, _, cb = ctx[b]
            ra = ca.isend_enqueue(src[a], S, mpix.MPI_BYTE, b, Ktag)
            rb = cb.irecv_enqueue(dst[b], S, mpix.MPI_BYTE, a, Ktag)
            if a == b:
                mpix.waitall_enqueue([ra, rb])
            else:
                mpix.wait_enqueue(ra)
                mpix.wait_enqueue(rb)

    def sync():
        for d in set(dev):
            torch.cuda.synchronize(d)

    log('correctness of the measured path (same inputs as the timed lo')
    # correctness of the measured path (same inputs as the timed loop)
    step()
    sync()
    for a, b in pairs:
        assert torch.equal(dst[b], src[a].to(dev[b])), "payload mismatch"

    clocks = ClockSampler(0)
    clocks.start()
    for _ in range(args.warmup):
        step()
    sync()
    log('soak so that the clock sampler sees the step under load (~0.5')
    # soak so that the clock sampler sees the step under load (~0.5 s)
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.5:
        for _ in range(10):
            step()
        sync()

    log('---- timed region: K steps, events on every stream, max over ')
    # ---- timed region: K steps, events on every stream, max over GPUs ----
    starts = {r: torch.cuda.Event(enable_timing=True) for r in range(P)}
    ends = {r: torch.cuda.Event(enable_timing=True) for r in range(P)}
    sync()
    l0 = mpix.launch_count()
    for r in range(P):
        starts[r].record(ctx[r][0])
    for k in range(args.steps):
        step()
    for r in range(P):
        ends[r].record(ctx[r][0])
    sync()
    launches = mpix.launch_count() - l0
    clk = clocks.stop()
    ms = max(starts[r].elapsed_time(ends[r]) for r in range(P))
    t_step = ms / 1e3 / args.steps
    value = S * len(pairs) / t_step / 1e9

    log('dominant kernel: the copy grid (k_gcopy), timed with CUDA eve')
    # dominant kernel: the copy grid (k_gcopy), timed with CUDA events the
    # runtime records around each launch on the launching stream
    # (MPIXT_Copy_timing; only grids that copied are counted), over K more
    # steps of the same workload
    mpix.testing.copy_timing(True)
    for k in range(args.steps):
        step()
    sync()
    tot_ms, ncopy, moved = mpix.testing.copy_timing_read()
    mpix.testing.copy_timing(False)
    k_ms = tot_ms / max(ncopy, 1)
    k_bytes = moved / max(ncopy, 1)  # message bytes one copying grid moved

    log('roofline of the dominant kernel (the copy grid that moves the')
    # roofline of the dominant kernel (the copy grid that moves the payload)
    if P == 1:
        alg_bytes = 2 * k_bytes  # read + write of the message on one GPU
        peak = pk.get("hbm_gbs", 6650.0)
        roof = {"bound": "hbm", "unit": "GB/s", "peak_source": "MEASURED_PEAKS.json hbm_gbs"
                if "hbm_gbs" in pk else "fallback 6650 GB/s (B200_PROFILING.md)"}
    else:
        alg_bytes = k_bytes
        peak = 770.0
        roof = {"bound": "nvlink", "unit": "GB/s",
                "peak_source": "measured peer copy 770 GB/s per direction (B200_PROFILING.md); "
                               "nominal 900"}
    achieved = alg_bytes / (k_ms / 1e3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if P == 1 and os.path.exists(tf):  # captured on the loopback workload
        try:
            traffic = json.load(open(tf)).get(f"p2p_recv_{S}")
        except Exception:
            traffic = None
    roof.update({"achieved": achieved, "peak": peak, "frac": achieved / peak, "traffic": traffic,
                 "kernel": "mpix::k_gcopy (the copy grid of the message; the second arriver's)",
                 "kernel_ms": k_ms, "kernel_launches_timed": ncopy,
                 "algorithmic_bytes_per_launch": alg_bytes,
                 "step_frac": (2 * S if P == 1 else S) * len(pairs) / t_step / 1e9 / peak,
                 **({} if P == 1 else {"frac_of_nominal_900": achieved / 900.0}),
                 "step_note": "whole step (all launches: post, decide, copy, complete, wait) "
                              "against the same roofline"})

    log('---- e2e through the C ABI with host buffers ----')
    # ---- e2e through the C ABI with host buffers ----
    e2e = e2e_pass(args, mpix, torch, ctx, pairs, src, dst, S)

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {
            "workload": ("loopback: Isend/Irecv/Waitall_enqueue self-message on one stream, 1 GPU"
                         if P == 1 else f"{len(pairs)} GPU pair(s), Isend/Irecv/Wait_enqueue"),
            "message_bytes": S, "ranks": P, "parallelism": "none (messaging runtime)",
            "l2": "inputs larger than L2 (src+dst = 2 x message > 126 MB)",
            "baseline_config": "BASELINE.json configs[1] at one GPU (SURVEY.md §8d cfg2)",
            **({"devices": dev, "note": "--share-gpus validation run, not a measurement"}
               if args.share_gpus else {}),
        },
        "roofline": roof,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
    }
    if not args.no_extras and P == 1:
        line["extras"] = extras(args, mpix, torch, w, ctx)
    if not args.no_extras and P > 1:
        line["extras"] = extras_ngpu(args, mpix, torch, w, ctx, dev)
    if rank0_cpu() and P == 1:  # the CPU baseline: rank 0 at N=1 only
        line["cpu_baseline"] = cpu_reference_selfmsg(S, args.cpu_seconds)
        if not args.no_extras:
            line["cpu_reference_configs"] = cpu_reference_configs()
    sync()
    w.finalize()
    if not args.no_extras and P == 1:
        line["extras"].update(extras_multirank(args, mpix, torch))
    return line


def rank0_cpu():
    return dist_env()[0] == 0


def e2e_pass(args, mpix, torch, ctx, pairs, src, dst, S):
    """Same metric through the public API with HOST buffers: per step the
    input message is copied H2D from pinned memory, sent/received through the
    enqueue calls, a consumer kernel checksums the delivered payload, and the
    8-byte checksum is read back on the host (stream synchronised)."""
    host = {a: torch.empty(S, dtype=torch.uint8, pin_memory=True) for a, _ in pairs}
    for a, _ in pairs:
        host[a].copy_(src[a].cpu())
    sums = {b: torch.zeros(1, dtype=torch.int64, device=dst[b].device) for _, b in pairs}
    hsum = {b: torch.zeros(1, dtype=torch.int64, pin_memory=True) for _, b in pairs}

    def one(tag):
        for a, b in pairs:
            sa, _, ca = ctx[a]
            sb, _, cb = ctx[b]
            with torch.cuda.stream(sa):
                src[a].copy_(host[a], non_blocking=True)
            ra = ca.isend_enqueue(src[a], S, mpix.MPI_BYTE, b, 30000 + tag)
            rb = cb.irecv_enqueue(dst[b], S, mpix.MPI_BYTE, a, 30000 + tag)
            if a == b:
                mpix.waitall_enqueue([ra, rb])
            else:
                mpix.wait_enqueue(ra)
                mpix.wait_enqueue(rb)
            mpix.testing.checksum(dst[b], S, sums[b], sb)
            with torch.cuda.stream(sb):
                hsum[b].copy_(sums[b], non_blocking=True)
        for a, b in pairs:
            ctx[a][0].synchronize()
            ctx[b][0].synchronize()

    for i in range(max(1, args.warmup)):
        one(i % 1000)
    t0 = time.perf_counter()
    for i in range(args.steps):
        one(i % 1000)
    t = time.perf_counter() - t0
    v = S * len(pairs) * args.steps / t / 1e9
    # the bound: the same H2D copy alone (pinned host -> device, synchronised)
    a0 = pairs[0][0]
    sa = ctx[a0][0]
    with torch.cuda.stream(sa):
        src[a0].copy_(host[a0], non_blocking=True)
    sa.synchronize()
    t1 = time.perf_counter()
    for _ in range(args.steps):
        with torch.cuda.stream(sa):
            src[a0].copy_(host[a0], non_blocking=True)
        sa.synchronize()
    h2d = S * args.steps / (time.perf_counter() - t1) / 1e9
    return {"value": v, "unit": "GB/s",
            "h2d_bytes_per_step": S * len(pairs), "d2h_bytes_per_step": 8 * len(pairs),
            "timing": "host wall clock, stream synchronised every step",
            "bound": {"pcie_h2d_GBps": h2d, "frac": v / (h2d * len(pairs)),
                      "note": "the step's H2D of the input dominates; same pinned copy timed alone"}}


def extras(args, mpix, torch, w, ctx):
    """Secondary measurements on the same GPU (not the headline)."""
    out = {}
    s0, _, c0 = ctx[0]
    big = torch.empty(1 << 30, dtype=torch.uint8, device=0)
    big2 = torch.empty(1 << 30, dtype=torch.uint8, device=0)

    log('launch floor: back-to-back empty kernels in one stream (nativ')
    # launch floor: back-to-back empty kernels in one stream (native loop)
    mpix.testing.empty_loop(50, s0)
    dev, host = mpix.testing.empty_loop(2000, s0)
    t_empty = dev / 2000
    out["launch_floor_us"] = t_empty * 1e6
    out["launch_floor_host_us"] = host / 2000 * 1e6

    log('loopback sweep (Isend/Irecv/Waitall on one stream, native loo')
    # loopback sweep (Isend/Irecv/Waitall on one stream, native loop)
    sweep = {}
    for sz in [8, 4096, 65536, 1 << 20, 16 << 20, 64 << 20, 256 << 20, 1 << 30]:
        it = 500 if sz <= (1 << 20) else (50 if sz <= (64 << 20) else 10)
        mpix.testing.loopback(c0, big, big2, sz, 5, s0)
        dev, host = mpix.testing.loopback(c0, big, big2, sz, it, s0)
        t = dev / it
        sweep[str(sz)] = {"us": t * 1e6, "host_us": host / it * 1e6, "GBps": sz / t / 1e9,
                          "hbm_frac": 2 * sz / t / 1e9 / peaks().get("hbm_gbs", 6650.0)}
    out["loopback_sweep"] = sweep

    log('in-stream latency: producer -> Send_enqueue -> Recv_enqueue -')
    # in-stream latency: producer -> Send_enqueue -> Recv_enqueue -> consumer
    # (8 B self message, one stream, native driver so the host runs ahead)
    prod = torch.zeros(2, dtype=torch.float32, device=0)
    cons = torch.zeros(2, dtype=torch.float32, device=0)
    mpix.testing.selfchain(c0, prod, cons, 2, 50, s0)
    dev, host = mpix.testing.selfchain(c0, prod, cons, 2, 1000, s0)
    out["inloop_self_chain_us"] = dev / 1000 * 1e6
    out["inloop_self_chain_host_us"] = host / 1000 * 1e6
    out["inloop_self_chain_over_floor_us"] = (dev / 1000 - 4 * t_empty) * 1e6
    return out


def extras_ngpu(args, mpix, torch, w, ctx, dev):
    """N > 1 (one rank per GPU): Allreduce_enqueue busbw over all N GPUs
    (BASELINE cfg3 at N), and Send/Recv_enqueue ping-pong latency between
    ranks 0 and 1 (cfg2 latency across NVLink)."""
    out = {}
    P = len(dev)
    cs = [ctx[r][2] for r in range(P)]
    ss = [ctx[r][0] for r in range(P)]
    ar = {}
    for name, tdt, mdt in (("f32", torch.float32, mpix.MPI_FLOAT), ("bf16", torch.bfloat16, mpix.MPIX_BFLOAT16)):
        nbytes = 256 << 20
        cnt = nbytes // torch.tensor([], dtype=tdt).element_size()
        sb = [torch.ones(cnt, dtype=tdt, device=dev[r]) for r in range(P)]
        rb = [torch.empty(cnt, dtype=tdt, device=dev[r]) for r in range(P)]
        mpix.testing.allreduce_loop(cs, ss, dev, sb, rb, cnt, mdt, 2)
        dev_s, _ = mpix.testing.allreduce_loop(cs, ss, dev, sb, rb, cnt, mdt, 10)
        for d in set(dev):
            torch.cuda.synchronize(d)
        t = dev_s / 10
        algbw = nbytes / t / 1e9
        ar[name] = {"ms": t * 1e3, "algbw_GBps": algbw, "busbw_GBps": algbw * 2 * (P - 1) / P,
                    "busbw_frac_of_770": algbw * 2 * (P - 1) / P / 770.0,
                    "check": float(rb[0][0]) == float(P)}
        del sb, rb
    out["allreduce_256MiB"] = ar
    pp = {}
    for nb in (8, 4096, 65536, 1 << 20, 64 << 20):
        b0 = torch.zeros(max(nb, 16), dtype=torch.uint8, device=dev[0])
        b1 = torch.zeros(max(nb, 16), dtype=torch.uint8, device=dev[1])
        iters = 200 if nb <= (1 << 20) else 20
        mpix.testing.pingpong(cs[0], cs[1], b0, b1, nb, 10, ss[0], ss[1], dev[0], dev[1])
        d, h = mpix.testing.pingpong(cs[0], cs[1], b0, b1, nb, iters, ss[0], ss[1], dev[0], dev[1])
        pp[str(nb)] = {"half_rtt_us": d / (2 * iters) * 1e6,
                       "GBps": nb / (d / (2 * iters)) / 1e9}
    out["pingpong_rank0_rank1"] = pp
    return out


def extras_multirank(args, mpix, torch):
    """cfg3 / cfg4 / cfg5 on the visible GPU(s); ranks share GPUs when fewer
    than 8 are visible (numbers are then HBM-bound, not NVLink-bound)."""
    from paper_2208_13707_b200.workloads import HaloStencil, msgrate
    out = {}
    ndev = torch.cuda.device_count()

    def world(P, priority=0):
        devs = [r % ndev for r in range(P)]
        w = mpix.World(P, devs)
        ctx = {}

        def setup(r):
            with torch.cuda.device(devs[r]):
                s = mpix.testing.new_stream(devs[r], priority)
            ctx[r] = (s, w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s)), devs[r])
        w.run_ranks(setup)
        return w, ctx

    def sync_all(ctx):
        for s, _, _ in ctx.values():
            s.synchronize()

    log('cfg2 latency: blocking Send/Recv_enqueue ping-pong between 2 ')
    # cfg2 latency: blocking Send/Recv_enqueue ping-pong between 2 ranks
    # (both on GPU 0 unless 2 GPUs are visible), half round trip
    w, ctx = world(2)
    pp = {}
    for nb in (8, 4096, 65536, 1 << 20):
        b0 = torch.zeros(max(nb, 16), dtype=torch.uint8, device=ctx[0][2])
        b1 = torch.zeros(max(nb, 16), dtype=torch.uint8, device=ctx[1][2])
        mpix.testing.pingpong(ctx[0][1], ctx[1][1], b0, b1, nb, 20, ctx[0][0], ctx[1][0],
                              ctx[0][2], ctx[1][2])
        iters = 500 if nb <= 65536 else 100
        dev, host = mpix.testing.pingpong(ctx[0][1], ctx[1][1], b0, b1, nb, iters, ctx[0][0],
                                          ctx[1][0], ctx[0][2], ctx[1][2])
        pp[str(nb)] = {"half_rtt_us": dev / (2 * iters) * 1e6,
                       "host_us_per_half_rtt": host / (2 * iters) * 1e6}
    sync_all(ctx)
    w.finalize()
    out["pingpong_2ranks"] = {"gpus": len({ctx[0][2], ctx[1][2]}), **pp}

    log('unpaired exchange: 2 ranks, 256 MiB each way, device handshake')
    # The headline's self-messages are host-paired (no descriptors, DESIGN.md
    # §3); this is the cross-rank device handshake (post, scan, second
    # arriver's copy grid, completion) on the same 256 MiB, both directions at
    # once: Isend + Irecv + Waitall_enqueue per rank and step.
    w, ctx = world(2)
    S = 256 << 20
    xs = [torch.empty(S, dtype=torch.uint8, device=ctx[r][2]) for r in range(2)]
    xd = [torch.empty(S, dtype=torch.uint8, device=ctx[r][2]) for r in range(2)]
    for r in range(2):
        xs[r].fill_(r + 1)
    torch.cuda.synchronize()

    X = (ctx[0][1], ctx[1][1], xs[0], xd[0], xs[1], xd[1], S)
    mpix.testing.exchange(*X, 3, ctx[0][0], ctx[1][0], ctx[0][2], ctx[1][2])
    K = 20
    t = mpix.testing.exchange(*X, K, ctx[0][0], ctx[1][0], ctx[0][2], ctx[1][2]) / K
    sync_all(ctx)
    ok = bool(int(xd[0][0]) == 2 and int(xd[1][-1]) == 1)
    gpus = len({ctx[0][2], ctx[1][2]})
    out["exchange_256MiB_2ranks_unpaired"] = {
        "gpus": gpus, "step_us": t * 1e6, "GBps_per_direction": S / t / 1e9,
        "GBps_both": 2 * S / t / 1e9,
        "hbm_frac_step": (4 * S / t / 1e9) / peaks().get("hbm_gbs", 6650.0) if gpus == 1 else None,
        "driver": "native threads over the C ABI (MPIXT_Exchange): per step each rank enqueues "
                  "Irecv + Isend + Waitall_enqueue",
        "note": "on one GPU both copies (2 x S of HBM traffic each) share HBM",
        "check": ok}
    del xs, xd
    w.finalize()

    log('cfg3: Allreduce_enqueue 256 MiB fp32 and bf16 at P = 1, 2, 4,')
    # cfg3: Allreduce_enqueue 256 MiB fp32 and bf16 at P = 1, 2, 4, 8
    ar = {}
    for P in (1, 2, 4, 8):
        w, ctx = world(P)
        for dt, tdt, mdt in (("f32", torch.float32, mpix.MPI_FLOAT), ("bf16", torch.bfloat16, mpix.MPIX_BFLOAT16)):
            nbytes = 256 << 20
            cnt = nbytes // torch.tensor([], dtype=tdt).element_size()
            sb = {r: torch.ones(cnt, dtype=tdt, device=ctx[r][2]) for r in range(P)}
            rb = {r: torch.empty(cnt, dtype=tdt, device=ctx[r][2]) for r in range(P)}
            iters = 10
            cs = [ctx[r][1] for r in range(P)]
            ss = [ctx[r][0] for r in range(P)]
            ds = [ctx[r][2] for r in range(P)]
            mpix.testing.allreduce_loop(cs, ss, ds, [sb[r] for r in range(P)],
                                        [rb[r] for r in range(P)], cnt, mdt, 2)
            dev_s, _ = mpix.testing.allreduce_loop(cs, ss, ds, [sb[r] for r in range(P)],
                                                   [rb[r] for r in range(P)], cnt, mdt, iters)
            sync_all(ctx)
            t = dev_s / iters
            algbw = nbytes / t / 1e9
            ar[f"{dt}_P{P}"] = {"ms": t * 1e3, "algbw_GBps": algbw,
                                "busbw_GBps": algbw * 2 * (P - 1) / P,
                                "ranks_per_gpu": -(-P // ndev),
                                "check": float(rb[0][0]) == float(P)}
            del sb, rb
        # small-message latency (one-shot <= 64 KiB), native driver
        if P in (2, 8):
            lat = {}
            for nbytes in (8, 4096, 65536, 1 << 20):
                cnt = max(1, nbytes // 4)
                sb = [torch.ones(cnt, dtype=torch.float32, device=ctx[r][2]) for r in range(P)]
                rb = [torch.empty(cnt, dtype=torch.float32, device=ctx[r][2]) for r in range(P)]
                cs = [ctx[r][1] for r in range(P)]
                ss = [ctx[r][0] for r in range(P)]
                ds = [ctx[r][2] for r in range(P)]
                mpix.testing.allreduce_loop(cs, ss, ds, sb, rb, cnt, mpix.MPI_FLOAT, 5)
                dev_s, host_s = mpix.testing.allreduce_loop(cs, ss, ds, sb, rb, cnt, mpix.MPI_FLOAT, 200)
                sync_all(ctx)
                lat[str(nbytes)] = {"us": dev_s / 200 * 1e6, "host_us": host_s / 200 * 1e6,
                                    "check": float(rb[0][0]) == float(P)}
            ar[f"latency_f32_P{P}"] = lat
        w.finalize()
    out["allreduce_256MiB"] = ar

    log('the other enqueued collectives at P = 8 (ranks share the visi')
    # the other enqueued collectives at P = 8 (ranks share the visible GPUs),
    # 256 MiB per rank of fp32: bcast of 256 MiB, allgather of 32 MiB blocks,
    # reduce_scatter_block of 32 MiB blocks (256 MiB input per rank)
    w, ctx = world(8)
    P8 = 8
    nb = 256 << 20
    cnt = nb // 4
    big = {r: torch.ones(cnt, dtype=torch.float32, device=ctx[r][2]) for r in range(P8)}
    small = {r: torch.ones(cnt // P8, dtype=torch.float32, device=ctx[r][2]) for r in range(P8)}
    big2 = {r: torch.empty(cnt, dtype=torch.float32, device=ctx[r][2]) for r in range(P8)}
    colls = {
        "bcast_256MiB": lambda r: ctx[r][1].bcast_enqueue(big[r], cnt, mpix.MPI_FLOAT, 0),
        "allgather_8x32MiB": lambda r: ctx[r][1].allgather_enqueue(small[r], big[r], cnt // P8,
                                                                   mpix.MPI_FLOAT),
        "reduce_scatter_8x32MiB": lambda r: ctx[r][1].reduce_scatter_block_enqueue(
            big[r], small[r], cnt // P8, mpix.MPI_FLOAT),
        "alltoall_8x32MiB": lambda r: ctx[r][1].alltoall_enqueue(big[r], big2[r], cnt // P8,
                                                                 mpix.MPI_FLOAT),
    }
    cres = {}
    for name, fn in colls.items():
        ev = {r: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for r in range(P8)}

        def loop(r, k, timed, fn=fn, ev=ev):
            if timed:
                ev[r][0].record(ctx[r][0])
            for _ in range(k):
                fn(r)
            if timed:
                ev[r][1].record(ctx[r][0])
        w.run_ranks(lambda r: loop(r, 1, False))
        sync_all(ctx)
        w.run_ranks(lambda r: loop(r, 5, True))
        sync_all(ctx)
        t = max(a.elapsed_time(b) for a, b in ev.values()) / 1e3 / 5
        # bytes every rank receives (the algorithmic per-rank volume)
        per_rank = {"bcast_256MiB": nb, "allgather_8x32MiB": nb * 7 // 8,
                    "reduce_scatter_8x32MiB": nb, "alltoall_8x32MiB": nb * 7 // 8}[name]
        cres[name] = {"ms": t * 1e3, "GBps_per_rank": per_rank / t / 1e9, "ranks_per_gpu": -(-P8 // ndev)}
    del big, small, big2
    w.finalize()
    out["collectives_P8"] = cres

    log('cfg5: 3-D halo stencil, 2x2x2 periodic, 512^3 fp32 per rank')
    # cfg5: 3-D halo stencil, 2x2x2 periodic, 512^3 fp32 per rank
    n = 512  # BASELINE cfg5: 512^3 fp32 per rank (8 ranks share the visible GPUs)
    log('communication streams above the default priority: the exchang')
    # communication streams above the default priority: the exchange's
    # handshake and copy kernels are scheduled ahead of the interior stencil
    # CTAs (on the default-priority second stream) they overlap with
    w, ctx = world(8, priority=-5)
    blocks = {r: HaloStencil(r, n, ctx[r][0], ctx[r][1], device=ctx[r][2]) for r in range(8)}
    w.run_ranks(lambda r: blocks[r].step())  # the Python step (pipelined), warm-up
    sync_all(ctx)
    devs8 = [ctx[r][2] for r in range(8)]
    T = mpix.testing
    halo = {"block": f"{n}^3 fp32 per rank, 8 ranks 2x2x2 periodic", "ranks_per_gpu": -(-8 // ndev),
            "face_bytes": n * n * 4, "driver": "native (one host thread per rank, MPIXT_Halo_steps)"}
    steps = 10
    for name, mode in (("seq", T.HALO_SEQ), ("pipe", T.HALO_PIPE), ("compute", T.HALO_COMPUTE),
                       ("exchange", T.HALO_EXCHANGE)):
        T.halo_steps(list(blocks.values()), 2, devs8, mode)
        d, h = T.halo_steps(list(blocks.values()), steps, devs8, mode)
        halo[f"{name}_step_ms"] = d / steps * 1e3
    t_seq, t_pipe = halo["seq_step_ms"], halo["pipe_step_ms"]
    t_comp, t_x = halo["compute_step_ms"], halo["exchange_step_ms"]
    log('stencil roofline: every rank reads u once and writes its n^3 ')
    # stencil roofline: every rank reads u once and writes its n^3 interior once
    sb = 8 * 2 * n ** 3 * 4
    halo["stencil_hbm_GBps"] = sb / (t_comp / 1e3) / 1e9 / max(1, ndev)
    halo["stencil_frac_of_hbm"] = halo["stencil_hbm_GBps"] / peaks().get("hbm_gbs", 6650.0)
    log('exposed communication and overlap efficiency (SURVEY.md §8(d)')
    # exposed communication and overlap efficiency:
    # the share of the exchange hidden behind the stencil
    halo["exposed_comm_ms_seq"] = t_seq - t_comp
    halo["exposed_comm_ms_pipe"] = t_pipe - t_comp
    halo["overlap_efficiency"] = max(0.0, min(1.0, 1 - (t_pipe - t_comp) / t_x)) if t_x > 0 else None
    out["halo3d"] = halo
    del blocks
    w.finalize()

    log('cfg4: 8 ranks x 4 stream comms, ring, 8-byte messages, window')
    # cfg4: 8 ranks x 4 stream comms, ring, 8-byte messages, window 64
    P, S, W, B = 8, 4, 64, 50
    devs = [r % ndev for r in range(P)]
    w = mpix.World(P, devs)
    ctxs = [[] for _ in range(P)]

    def setup(r):
        for k in range(S):
            with torch.cuda.device(devs[r]):
                s = mpix.testing.new_stream(devs[r])
            ctxs[r].append((s, w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s))))
    w.run_ranks(setup)
    bufs = [[(torch.zeros(2, dtype=torch.int32, device=devs[r]),
              torch.zeros((W, 2), dtype=torch.int32, device=devs[r])) for _ in range(S)] for r in range(P)]
    log('host-bound (enqueue threads): warm up twice, report the media')
    # host-bound (enqueue threads): warm up twice, report the median of 3 runs
    msgrate(w, ctxs, S, W, 1, bufs)
    for _ in range(2):
        msgrate(w, ctxs, S, W, B, bufs)
    runs = sorted((msgrate(w, ctxs, S, W, B, bufs) for _ in range(3)), key=lambda x: x["msgs_per_s"])
    res = dict(runs[1])
    res["runs_msgs_per_s"] = [x["msgs_per_s"] for x in runs]
    for d in range(ndev):
        torch.cuda.synchronize(d)
    out["msgrate_8B"] = {"ranks": P, "streams_per_rank": S, "window": W, **res,
                         "driver": "native C++ threads over the C ABI (MPIXT_Msgrate)",
                         "launches_per_window": "1 coalesced k_batch (2W = 128 operations + the Waitall)"}
    w.finalize()

    log('the same under the dynamic (wildcard-capable) matching engine')
    # the same under the dynamic (wildcard-capable) matching engine
    prev = os.environ.get("MPIX_MATCHING")
    os.environ["MPIX_MATCHING"] = "dynamic"
    try:
        w = mpix.World(P, devs)
        ctxs = [[] for _ in range(P)]
        w.run_ranks(setup)
        msgrate(w, ctxs, S, W, 1, bufs)
        res = msgrate(w, ctxs, S, W, B, bufs)
        for d in range(ndev):
            torch.cuda.synchronize(d)
        out["msgrate_8B_dynamic_matching"] = {"ranks": P, "streams_per_rank": S, "window": W, **res}
        w.finalize()
    finally:
        if prev is None:
            os.environ.pop("MPIX_MATCHING", None)
        else:
            os.environ["MPIX_MATCHING"] = prev

    log('paper Fig. 3: lock regimes over conventional p2p (2 ranks x T threads)')
    from paper_2208_13707_b200.workloads import fig3
    f3 = {}
    for regime, name in ((0, "global"), (1, "pervci"), (2, "stream")):
        f3[name] = {}
        for T in (1, 2, 4, 8):
            fig3(T, W=64, batches=5, regime=regime, torch=torch)  # warm-up
            f3[name][str(T)] = fig3(T, W=64, batches=50, regime=regime, torch=torch)["msgs_per_s"]
    out["fig3_lock_regimes_msgs_per_s"] = {
        "rates": f3, "messages_per_thread": 64 * 50, "bytes": 8,
        "driver": "native threads over the C ABI (MPIXT_Fig3), conventional MPI_Isend/Irecv/Waitall "
                  "+ credit, host wall clock as the reference (bench.cpp:200-223)"}
    log('CUDA-Graph capture: the same latency-bound patterns enqueued ')
    # CUDA-Graph capture: the same latency-bound patterns enqueued eagerly
    # from Python vs captured once and replayed (graph-capturable comms)
    from paper_2208_13707_b200.workloads import graph_latency
    out["graph_replay"] = graph_latency()
    return out


def main():
    # a stalled run prints every thread's stack (stderr) instead of dying silently
    import faulthandler
    faulthandler.dump_traceback_later(240, repeat=True, file=sys.stderr)
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_mpix(args)


if __name__ == "__main__":
    main()
