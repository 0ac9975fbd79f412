# final-kernel ncu evidence: launch lists + full captures (tools/profile_round.sh), tiny-window capture
O=gpurun_out/r02aa
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
bash tools/profile_round.sh $O/prof > $O/prof.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_batch_tiny -s 3 -c 1 -o $O/ktiny python tools/profile_loopback.py --size 8 --steps 5 --warmup 3 --window 32 > /dev/null 2>&1
ncu -i $O/ktiny.ncu-rep --page details --csv > $O/prof/k_batch_tiny_window32_details.csv 2>/dev/null
ncu -i $O/ktiny.ncu-rep --page raw --csv > $O/prof/k_batch_tiny_window32_raw.csv 2>/dev/null
rm -f $O/ktiny.ncu-rep
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/prof/smoke_ncu_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_ncu.txt 2>&1
