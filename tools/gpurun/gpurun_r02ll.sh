# same-box A/B: k_op1 (MPIX_OP1=1) vs k_batch_tiny for single blocking operations
O=gpurun_out/r02ll
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
for i in 1 2; do
for op1 in 0 1; do
  echo "== MPIX_OP1=$op1" >> $O/ab.txt
  MPIX_OP1=$op1 timeout 120 python tools/pingpong_probe.py >> $O/ab.txt 2>&1
  MPIX_OP1=$op1 MPIX_FORCE_SYS=1 timeout 120 python tools/pingpong_probe.py >> $O/ab.txt 2>&1
done
done
timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_ll.py tests/test_gpu_model_check.py tests/test_gpu_conventional.py -q -x --timeout 200 -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
