# relaxed polling + register snapshots: full suite, stress modes, bench
O=gpurun_out/r02w8
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 1800 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for mode in "MPIX_FORCE_SYS=1" "MPIX_BATCH=0" "MPIX_LL=0" "MPIX_GRAPH=1" "MPIX_MATCHING=dynamic" "MPIX_CONV_BATCH=0"; do
  timeout 900 env $mode python -m pytest tests/test_gpu_p2p.py tests/test_gpu_batch.py tests/test_gpu_model_check.py tests/test_gpu_conventional.py tests/test_gpu_errors.py -q --timeout 200 -p no:cacheprovider > $O/pytest_$mode.txt 2>&1; echo "rc=$?" >> $O/pytest_$mode.txt
done
timeout 900 env MPIX_SPIN_TIMEOUT_MS=30000 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
