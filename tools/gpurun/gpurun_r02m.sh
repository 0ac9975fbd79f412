# round 2, call m: LL + polling receives + k_batch_tiny: full GPU suite, stress modes, bench
O=gpurun_out/r02m
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 200 -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 600 env MPIX_FORCE_SYS=1 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_batch.py tests/test_gpu_model_check.py tests/test_gpu_graph.py tests/test_gpu_conventional.py -q -x --timeout 200 -p no:cacheprovider > $O/pytest_sys.txt 2>&1; echo "rc=$?" >> $O/pytest_sys.txt
timeout 600 env MPIX_BATCH=0 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_batch.py tests/test_gpu_model_check.py -q -x --timeout 200 -p no:cacheprovider > $O/pytest_nobatch.txt 2>&1; echo "rc=$?" >> $O/pytest_nobatch.txt
timeout 600 env MPIX_LL=0 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_batch.py tests/test_gpu_model_check.py -q -x --timeout 200 -p no:cacheprovider > $O/pytest_noll.txt 2>&1; echo "rc=$?" >> $O/pytest_noll.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
