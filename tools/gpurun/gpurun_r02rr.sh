# LL-eager: the full suite twice + stress modes
O=gpurun_out/r02rr2
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
for i in 1 2; do
  timeout 1800 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider > $O/pytest$i.txt 2>&1; echo "rc=$?" >> $O/pytest$i.txt
done
for mode in "MPIX_FORCE_SYS=1" "MPIX_BATCH=0" "MPIX_GRAPH=1" "MPIX_MATCHING=dynamic"; do
  timeout 900 env $mode python -m pytest tests/test_gpu_p2p.py tests/test_gpu_batch.py tests/test_gpu_model_check.py tests/test_gpu_conventional.py tests/test_gpu_errors.py tests/test_gpu_ll.py -q --timeout 200 -p no:cacheprovider > $O/pytest_$mode.txt 2>&1; echo "rc=$?" >> $O/pytest_$mode.txt
done
