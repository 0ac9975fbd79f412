O=gpurun_out/r02r
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 1800 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for i in 1 2 3; do timeout 900 env MPIX_SPIN_TIMEOUT_MS=30000 python bench.py > $O/bench$i.json 2> $O/bench$i.err; echo "rc=$?" >> $O/bench$i.err; done
timeout 120 python tools/pingpong_probe.py > $O/pingpong.txt 2>&1
timeout 120 env MPIX_FORCE_SYS=1 python tools/pingpong_probe.py >> $O/pingpong.txt 2>&1
bash tools/gpurun/gpurun_r02p.sh
