O=gpurun_out/r02h
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 120 python tools/trace_pingpong.py 8 400 > $O/trace_pp.txt 2>&1
timeout 120 env MPIX_FORCE_SYS=1 python tools/trace_pingpong.py 8 400 >> $O/trace_pp.txt 2>&1
timeout 120 python tools/trace_small.py 8 > $O/trace_small.txt 2>&1
timeout 120 python tools/graph_loopback.py > $O/graph_loopback.txt 2>&1
