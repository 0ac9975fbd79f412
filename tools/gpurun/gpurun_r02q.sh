O=gpurun_out/r02q
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 300 python -m pytest tests/test_gpu_fig3.py -q -x --timeout 120 -p no:cacheprovider > $O/pytest_fig3.txt 2>&1; echo "rc=$?" >> $O/pytest_fig3.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 900 env MPIX_SPIN_TIMEOUT_MS=30000 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 1500 bash tools/sanitize.sh $O/sanitize > $O/sanitize.log 2>&1
bash tools/gpurun/gpurun_r02p.sh
