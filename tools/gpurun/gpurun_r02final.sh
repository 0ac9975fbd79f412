# final evidence: suite + stress + bench + smoke (tools/gpurun/gpurun_r02w.sh), probes, ncu
bash tools/gpurun/gpurun_r02w.sh
O=gpurun_out/r02w8
export CUDA_MODULE_LOADING=EAGER
timeout 120 python tools/pingpong_probe.py > $O/pp.txt 2>&1
timeout 120 env MPIX_FORCE_SYS=1 python tools/pingpong_probe.py >> $O/pp.txt 2>&1
timeout 120 python tools/graph_loopback.py >> $O/pp.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/smoke_ncu.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_ncu.txt 2>&1; echo "rc=$?" >> $O/smoke_ncu.txt
timeout 1200 bash tools/profile_round.sh $O/prof > $O/prof.log 2>&1
