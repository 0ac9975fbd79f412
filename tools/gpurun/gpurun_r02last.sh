# last call of the round: smoke (plain and under ncu), bench N=1, reference arm, probe
O=gpurun_out/r02last
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/smoke_ncu.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_ncu.txt 2>&1; echo "rc=$?" >> $O/smoke_ncu.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 120 python tools/pingpong_probe.py > $O/pp.txt 2>&1
timeout 120 env MPIX_FORCE_SYS=1 python tools/pingpong_probe.py >> $O/pp.txt 2>&1
