# round 2, call b: suite + smoke (plain and under ncu) + stencil probe + bench + memop probe
set -x
O=gpurun_out/r02b
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 150 env MPIX_SPIN_TIMEOUT_MS=3000 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/smoke_ncu.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_ncu.txt 2>&1; echo "rc=$?" >> $O/smoke_ncu.txt
timeout 120 tools/stencil_probe 512 10 > $O/stencil_probe.txt 2>&1; echo "rc=$?" >> $O/stencil_probe.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 150 -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 60 tools/memop_probe lat > $O/memop_lat.txt 2>&1; echo "rc=$?" >> $O/memop_lat.txt
timeout 90 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/memop_serial_ncu.csv tools/memop_probe serial 300 > $O/memop_serial_ncu.txt 2>&1; echo "rc=$?" >> $O/memop_serial_ncu.txt
