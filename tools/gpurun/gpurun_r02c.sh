# round 2, call c: smoke under ncu (co-residency probe), fixed batching rule, pipelined halo, stencil shapes, latency probes, bench
set -x
O=gpurun_out/r02c
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/smoke_ncu.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_ncu.txt 2>&1; echo "rc=$?" >> $O/smoke_ncu.txt
timeout 120 tools/stencil_probe 512 10 > $O/stencil_probe.txt 2>&1; echo "rc=$?" >> $O/stencil_probe.txt
timeout 1200 python -m pytest tests/test_gpu_batch.py tests/test_gpu_model_check.py tests/test_gpu_workloads.py tests/test_gpu_robust.py -q --timeout 300 -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 120 python tools/trace_small.py 8 > $O/trace_small.txt 2>&1
timeout 120 python tools/pingpong_probe.py > $O/pingpong.txt 2>&1
timeout 120 env MPIX_FORCE_SYS=1 python tools/pingpong_probe.py >> $O/pingpong.txt 2>&1
timeout 60 tools/memop_probe lat 3 > $O/memop_lat.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
