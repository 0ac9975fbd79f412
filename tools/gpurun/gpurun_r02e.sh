# round 2, call e: latency floors and the ping-pong phase breakdown
O=gpurun_out/r02e
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 120 tools/memop_probe lat > $O/memop_lat.txt 2>&1
timeout 120 python tools/trace_pingpong.py 8 400 > $O/trace_pp.txt 2>&1
timeout 120 env MPIX_FORCE_SYS=1 python tools/trace_pingpong.py 8 400 >> $O/trace_pp.txt 2>&1
timeout 120 python tools/pingpong_probe.py > $O/pingpong.txt 2>&1
timeout 120 env MPIX_FORCE_SYS=1 python tools/pingpong_probe.py >> $O/pingpong.txt 2>&1
timeout 120 python tools/trace_small.py 8 > $O/trace_small.txt 2>&1
