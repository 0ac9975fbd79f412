# round 2, call f: latency A/B (noinline protocol paths)
O=gpurun_out/r02f
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 120 python tools/trace_pingpong.py 8 400 > $O/trace_pp.txt 2>&1
timeout 120 env MPIX_FORCE_SYS=1 python tools/trace_pingpong.py 8 400 >> $O/trace_pp.txt 2>&1
timeout 120 python tools/pingpong_probe.py > $O/pingpong.txt 2>&1
timeout 120 env MPIX_FORCE_SYS=1 python tools/pingpong_probe.py >> $O/pingpong.txt 2>&1
timeout 120 python tools/trace_small.py 8 > $O/trace_small.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_batch.py -q -x --timeout 120 -p no:cacheprovider > $O/pytest.txt 2>&1
