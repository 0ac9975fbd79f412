O=gpurun_out/r02v
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 120 python tools/pingpong_probe.py > $O/pingpong.txt 2>&1
timeout 120 env MPIX_FORCE_SYS=1 python tools/pingpong_probe.py >> $O/pingpong.txt 2>&1
timeout 120 python tools/graph_loopback.py >> $O/pingpong.txt 2>&1
timeout 120 python tools/trace_small.py 8 >> $O/pingpong.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_batch.py tests/test_gpu_model_check.py tests/test_gpu_allreduce.py tests/test_gpu_collectives.py -q -x --timeout 200 -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
