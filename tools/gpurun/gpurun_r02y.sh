O=gpurun_out/r02y
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 120 python tools/trace_pingpong.py 8 400 > $O/tpp_pdl1.txt 2>&1
timeout 120 env MPIX_PDL=0 python tools/trace_pingpong.py 8 400 > $O/tpp_pdl0.txt 2>&1
timeout 120 python tools/pingpong_probe.py > $O/pp.txt 2>&1
timeout 120 env MPIX_PDL=0 python tools/pingpong_probe.py >> $O/pp.txt 2>&1
