set -x
mkdir -p gpurun_out/r02a
O=gpurun_out/r02a
nvidia-smi -L > $O/smi.txt
nproc > $O/nproc.txt; taskset -pc $$ >> $O/nproc.txt
tools/memop_probe lat > $O/memop_lat.txt 2>&1
timeout 90 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/memop_serial_ncu.csv tools/memop_probe serial 300 > $O/memop_serial_ncu.txt 2>&1; echo "rc=$?" >> $O/memop_serial_ncu.txt
timeout 150 env MPIX_SPIN_TIMEOUT_MS=3000 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/smoke_ncu.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_ncu.txt 2>&1; echo "rc=$?" >> $O/smoke_ncu.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
