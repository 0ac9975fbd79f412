#!/bin/bash
# ncu evidence for profiles/: launch lists (per-launch device time, cold and
# serialised) and one full capture per hot kernel. Run on the GPU box:
#   bash tools/profile_round.sh <outdir>
set -u
OUT=${1:-gpurun_out/prof}
mkdir -p "$OUT"
NCU="ncu --clock-control none"
# 1) launch list of the bench's N=1 step (256 MiB loopback)
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file "$OUT/launches_loopback_256MiB.csv" python tools/profile_loopback.py --steps 5 --warmup 3 > /dev/null 2>&1
# 2) launch list of 8-byte loopback windows (coalesced k_batch)
$NCU --metrics gpu__time_duration.sum --csv --log-file "$OUT/launches_window_8B.csv" \
  python tools/profile_loopback.py --size 8 --steps 5 --warmup 3 --window 32 > /dev/null 2>&1
# 3) full capture of the payload copy of one loopback step (the grouped copy
#    grid of the paired send/receive)
$NCU --set full --import-source on -k regex:k_gcopy -s 3 -c 1 -o "$OUT/k_gcopy" \
  python tools/profile_loopback.py --steps 5 --warmup 3 > /dev/null 2>&1
ncu -i "$OUT/k_gcopy.ncu-rep" --page raw --csv > "$OUT/k_gcopy_raw.csv" 2>/dev/null
ncu -i "$OUT/k_gcopy.ncu-rep" --page details --csv > "$OUT/k_gcopy_details.csv" 2>/dev/null
# 4) full capture of one coalesced window kernel (32 Isend + 32 Irecv + Waitall)
$NCU --set full --import-source on -k regex:k_batch -s 3 -c 1 -o "$OUT/k_batch" \
  python tools/profile_loopback.py --size 8 --steps 5 --warmup 3 --window 32 > /dev/null 2>&1
ncu -i "$OUT/k_batch.ncu-rep" --page details --csv > "$OUT/k_batch_details.csv" 2>/dev/null
# 5) allreduce reduce stage (P=4 buffers of 256 MiB bf16 on one GPU, two-shot share of rank 0)
$NCU --set full --import-source on -k regex:k_ar_reduce -s 4 -c 1 -o "$OUT/k_ar_reduce" \
  python tools/profile_allreduce.py --P 4 --reduce-only > /dev/null 2>&1
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file "$OUT/launches_reduce_only.csv" python tools/profile_allreduce.py --P 4 --reduce-only --iters 3 > /dev/null 2>&1
ncu -i "$OUT/k_ar_reduce.ncu-rep" --page raw --csv > "$OUT/k_ar_reduce_raw.csv" 2>/dev/null
ncu -i "$OUT/k_ar_reduce.ncu-rep" --page details --csv > "$OUT/k_ar_reduce_details.csv" 2>/dev/null
# keep the CSV exports only: the reports would overflow gpurun_out's 64 MiB
for rep in "$OUT"/k_gcopy.ncu-rep "$OUT"/k_batch.ncu-rep "$OUT"/k_ar_reduce.ncu-rep; do
  [ -f "$rep" ] && mv "$rep" /tmp/
done
ls -la "$OUT"
