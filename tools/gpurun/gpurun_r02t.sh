# conventional batching: conventional/multiplex/fig3 tests + full suite + fig3 A/B
O=gpurun_out/r02t
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 1800 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 600 python - > $O/fig3.txt 2>&1 <<'PY'
import os, json
from paper_2208_13707_b200.workloads import fig3
for cb in ("1", "0"):
    os.environ["MPIX_CONV_BATCH"] = cb
    res = {}
    for regime in (0, 1, 2):
        for T in (1, 4, 8):
            fig3(T, W=64, batches=5, regime=regime)
            res[f"{regime}/{T}"] = round(fig3(T, W=64, batches=50, regime=regime)["msgs_per_s"])
    print("conv_batch", cb, json.dumps(res), flush=True)
PY
bash tools/gpurun/gpurun_r02s.sh
