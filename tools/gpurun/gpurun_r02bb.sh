O=gpurun_out/r02bb
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 900 python -m pytest tests/test_gpu_wildcard.py tests/test_gpu_conventional.py tests/test_gpu_paths.py -q -x --timeout 200 -p no:cacheprovider > $O/pytest_dyn.txt 2>&1; echo "rc=$?" >> $O/pytest_dyn.txt
timeout 900 env MPIX_MATCHING=dynamic python -m pytest tests/test_gpu_p2p.py tests/test_gpu_batch.py tests/test_gpu_model_check.py tests/test_gpu_conventional.py tests/test_gpu_errors.py tests/test_gpu_workloads.py -q -x --timeout 200 -p no:cacheprovider > $O/pytest_dynmode.txt 2>&1; echo "rc=$?" >> $O/pytest_dynmode.txt
timeout 300 python - > $O/msgrate_dyn.txt 2>&1 <<'PY'
import os
os.environ["MPIX_MATCHING"] = "dynamic"
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch
from paper_2208_13707_b200 import mpix
from paper_2208_13707_b200.workloads import msgrate
P, S, W, B = 8, 4, 64, 50
w = mpix.World(P, [0] * P)
ctxs = [[] for _ in range(P)]
def setup(r):
    for k in range(S):
        s = mpix.testing.new_stream(0)
        ctxs[r].append((s, w.comm(r).stream_comm_create(mpix.Stream.from_cuda(s))))
w.run_ranks(setup)
bufs = [[(torch.zeros(2, dtype=torch.int32, device=0), torch.zeros((W, 2), dtype=torch.int32, device=0)) for _ in range(S)] for r in range(P)]
msgrate(w, ctxs, S, W, 1, bufs)
for _ in range(2): msgrate(w, ctxs, S, W, B, bufs)
print([round(msgrate(w, ctxs, S, W, B, bufs)["msgs_per_s"] / 1e6, 2) for _ in range(3)])
w.finalize()
PY
