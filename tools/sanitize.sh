#!/bin/bash
# Sanitizer pass over the enqueue path. Run on the GPU box:
#   bash tools/sanitize.sh <outdir>
# compute-sanitizer (memcheck, racecheck, synccheck) on the one-rank cases,
# ThreadSanitizer on the host runtime (libmpix_tsan.so) with two rank threads.
set -u
OUT=${1:-gpurun_out/sanitize}
mkdir -p "$OUT"
export CUDA_MODULE_LOADING=EAGER
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py --ranks 1 \
    > "$OUT/cs_$tool.txt" 2>&1
  echo "rc=$?" >> "$OUT/cs_$tool.txt"
done
if [ -f paper_2208_13707_b200/libmpix_tsan.so ]; then
  TSAN_OPTIONS="halt_on_error=0 report_signal_unsafe=0 second_deadlock_stack=1" \
    LD_PRELOAD=$(gcc -print-file-name=libtsan.so) MPIX_LIB_PATH=$PWD/paper_2208_13707_b200/libmpix_tsan.so \
    timeout 900 python tools/sanitize_cases.py --ranks 2 > "$OUT/tsan.txt" 2>&1
  echo "rc=$?" >> "$OUT/tsan.txt"
fi
tail -n 3 "$OUT"/*.txt
