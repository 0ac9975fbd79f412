"""Where the ping-pong half round trip goes (MPIX_TRACE=1: one k_proto per
operation, batching off). Two ranks on GPU 0, native blocking ping-pong;
every kernel stamps globaltimer at entry (g0 = t[0]), after the first scan
or poll hit (t[1]; an LL send posts right after it), after the decision
(t[2]), after the rescan (t[3]), before/after the completion stores (t[4],
t[5]) and at exit (g1).
  python tools/trace_pingpong.py [bytes] [iters]   (MPIX_FORCE_SYS=1: system scope)"""
import os
import statistics as st
import sys

os.environ["MPIX_TRACE"] = "1"
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_13707_b200 import mpix  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 8
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 400
w = mpix.World(2, [0, 0])
ctx = {}


def setup(r):
    s = mpix.testing.new_stream(0)
    ctx[r] = (s, w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s)))


w.run_ranks(setup)
b0 = torch.zeros(max(nb, 16), dtype=torch.uint8, device=0)
b1 = torch.zeros(max(nb, 16), dtype=torch.uint8, device=0)
d, h = mpix.testing.pingpong(ctx[0][1], ctx[1][1], b0, b1, nb, iters, ctx[0][0], ctx[1][0])
torch.cuda.synchronize()
half = d / iters / 2 * 1e6
A = sorted(mpix.trace_read(0, 4096), key=lambda r: r["seq"])
B = sorted(mpix.trace_read(1, 4096), key=lambda r: r["seq"])
# rank 0: send(i), recv(i); rank 1: recv(i), send(i)
n = min(len(A), len(B)) // 2
med = lambda xs: round(st.median(xs), 0) if xs else None
rows = {"A.send": [], "A.recv": [], "B.recv": [], "B.send": []}
x = {k: [] for k in ("A.send kernel", "A.send scan (g0->t1)", "A.send decide", "A.send fin",
                     "B.recv hit after A.send t1", "B.recv hit -> exit", "B.recv sees done after A.send fin",
                     "B recv->send gap", "B.send kernel", "B.send decide", "A.recv sees done after B.send fin",
                     "A send->recv gap", "A.recv posted (decide+rescan)", "half RTT (A.send g0 -> B.send g0)")}
acts = {}
for i in range(n // 4, n - 1):
    As, Ar = A[2 * i], A[2 * i + 1]
    Br, Bs = B[2 * i], B[2 * i + 1]
    if As["is_recv"] or not Ar["is_recv"] or not Br["is_recv"] or Bs["is_recv"]:
        continue
    acts[(As["action"], Ar["action"], Br["action"], Bs["action"])] = acts.get(
        (As["action"], Ar["action"], Br["action"], Bs["action"]), 0) + 1
    x["A.send kernel"].append(As["g1"] - As["g0"])
    x["A.send scan (g0->t1)"].append(As["t"][1] - As["g0"])
    x["A.send decide"].append(As["t"][3] - As["g0"])
    x["B.recv hit after A.send t1"].append(Br["t"][1] - As["t"][1])
    x["B.recv hit -> exit"].append(Br["g1"] - Br["t"][1])
    if As["t"][5]:
        x["A.send fin"].append(As["t"][5] - As["t"][4])
        x["B.recv sees done after A.send fin"].append(Br["g1"] - As["t"][5])
    x["B recv->send gap"].append(Bs["g0"] - Br["g1"])
    x["B.send kernel"].append(Bs["g1"] - Bs["g0"])
    x["B.send decide"].append(Bs["t"][3] - Bs["g0"])
    if Bs["t"][5]:
        x["A.recv sees done after B.send fin"].append(Ar["g1"] - Bs["t"][5])
    x["A send->recv gap"].append(Ar["g0"] - As["g1"])
    x["A.recv posted (decide+rescan)"].append(Ar["t"][3] - Ar["g0"])
    x["half RTT (A.send g0 -> B.send g0)"].append(Bs["g0"] - As["g0"])
import collections
print("SMs of A.send kernels:", collections.Counter(A[2 * i]["gt"][0] for i in range(n)).most_common(8))
print("SMs of B.recv kernels:", collections.Counter(B[2 * i]["gt"][0] for i in range(n)).most_common(8))
print("scope", "sys" if os.environ.get("MPIX_FORCE_SYS") == "1" else "gpu", "bytes", nb,
      "half RTT (event-timed) us", round(half, 2))
print("actions (A.send, A.recv, B.recv, B.send):", acts)
for k, v in x.items():
    print(f"  {k:45s} {med(v)} ns")
for r in range(2):
    ctx[r][0].synchronize()
w.finalize()
