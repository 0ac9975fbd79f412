O=gpurun_out/r02cc
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
for tw in 1 16 1 16; do
  echo "TINY_WARPS=$tw" >> $O/pp.txt
  timeout 120 env MPIX_TINY_WARPS=$tw python tools/pingpong_probe.py >> $O/pp.txt 2>&1
  timeout 120 env MPIX_TINY_WARPS=$tw MPIX_FORCE_SYS=1 python tools/pingpong_probe.py >> $O/pp.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_batch.py tests/test_gpu_model_check.py tests/test_gpu_conventional.py -q -x --timeout 200 -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
