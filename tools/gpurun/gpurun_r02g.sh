# round 2, call g: LL small sends + polling blocking receives: latency + full GPU suite
O=gpurun_out/r02g
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 120 python tools/trace_pingpong.py 8 400 > $O/trace_pp.txt 2>&1
timeout 120 env MPIX_FORCE_SYS=1 python tools/trace_pingpong.py 8 400 >> $O/trace_pp.txt 2>&1
timeout 120 python tools/pingpong_probe.py > $O/pingpong.txt 2>&1
timeout 120 env MPIX_FORCE_SYS=1 python tools/pingpong_probe.py >> $O/pingpong.txt 2>&1
timeout 120 env MPIX_LL=0 python tools/pingpong_probe.py >> $O/pingpong.txt 2>&1
timeout 120 env MPIX_LL=0 MPIX_FORCE_SYS=1 python tools/pingpong_probe.py >> $O/pingpong.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 200 -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
