O=gpurun_out/r02z
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 120 python tools/pingpong_probe.py > $O/pingpong.txt 2>&1
timeout 120 env MPIX_FORCE_SYS=1 python tools/pingpong_probe.py >> $O/pingpong.txt 2>&1
timeout 120 python tools/graph_loopback.py >> $O/pingpong.txt 2>&1
timeout 120 python tools/graph_loopback.py --graph 0 >> $O/pingpong.txt 2>&1
timeout 120 python tools/trace_pingpong.py 8 400 > $O/tpp.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_batch.py tests/test_gpu_model_check.py tests/test_gpu_graph.py tests/test_gpu_conventional.py -q -x --timeout 200 -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
