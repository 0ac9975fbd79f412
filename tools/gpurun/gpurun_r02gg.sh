O=gpurun_out/r02gg
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 120 python tools/graph_loopback.py > $O/g.txt 2>&1
timeout 120 python tools/graph_loopback.py --size 4096 >> $O/g.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_ll.py -q -x --timeout 200 -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 900 env MPIX_GRAPH=1 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_batch.py tests/test_gpu_model_check.py tests/test_gpu_ll.py -q -x --timeout 200 -p no:cacheprovider > $O/pytest_graph.txt 2>&1; echo "rc=$?" >> $O/pytest_graph.txt
