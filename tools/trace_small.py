"""Phase timing of the 1-CTA handshake kernels (MPIX_TRACE=1), loopback."""
import os, sys, statistics as st
os.environ["MPIX_TRACE"] = "1"
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2208_13707_b200 import mpix
S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
w = mpix.World(1, [0]); s = mpix.testing.new_stream(0)
c = w.comm(0).stream_comm_create(mpix.Stream.from_cuda(s))
src = torch.ones(max(S, 1), dtype=torch.uint8, device=0); dst = torch.zeros(max(S, 1), dtype=torch.uint8, device=0)
for i in range(50):
    r1 = c.isend_enqueue(src, S, 1, 0, 1); r2 = c.irecv_enqueue(dst, S, 1, 0, 1); mpix.waitall_enqueue([r1, r2])
torch.cuda.synchronize()
recs = mpix.trace_read(0)[20:]
for kind in (0, 1):
    rs = [r for r in recs if r["is_recv"] == kind]
    d = lambda a, b: st.median((r["t"][b] - r["t"][a]) for r in rs if r["t"][b] and r["t"][a])
    ph = ["scan1", "post", "rescan/cas", "copy", "fin"]
    out = {}
    for k in range(1, 6):
        try:
            out[ph[k - 1]] = round(d(k - 1, k), 0)
        except Exception:
            pass
    print("recv" if kind else "send", "ns per phase", out, "kernel ns", st.median(r["g1"] - r["g0"] for r in rs))
gaps = [recs[i + 1]["g0"] - recs[i]["g1"] for i in range(len(recs) - 1)]
print("gap between consecutive op kernels (ns, median)", st.median(gaps))
w.finalize()
