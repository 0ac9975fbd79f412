#!/bin/bash
# Repeat the handshake-heavy GPU tests under every protocol mode (races that
# need a rare interleaving show up as a watchdog error or a payload mismatch).
set -u
OUT=${1:-gpurun_out/stress.log}
: > "$OUT"
F="tests/test_gpu_p2p.py tests/test_gpu_batch.py tests/test_gpu_paths.py tests/test_gpu_staging.py tests/test_gpu_wildcard.py tests/test_gpu_allreduce.py tests/test_gpu_graph.py tests/test_gpu_ll.py tests/test_gpu_conventional.py tests/test_gpu_model_check.py"
for it in ${ITERS:-1 2 3}; do
  for mode in "" "MPIX_FORCE_SYS=1" "MPIX_GRAPH=1" "MPIX_MATCHING=dynamic" "MPIX_BATCH=0"; do
    r=$(env $mode timeout 900 python -m pytest $F -q -x --timeout 120 -p no:cacheprovider 2>&1 | tail -1)
    echo "iter $it mode [${mode:-default}]: $r" >> "$OUT"
  done
done
cat "$OUT"
