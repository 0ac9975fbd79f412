mkdir -p gpurun_out/r02qq
export CUDA_MODULE_LOADING=EAGER MPIX_SPIN_TIMEOUT_MS=15000
for lib in libmpix_old.so libmpix.so libmpix_old.so libmpix.so; do
  echo "== $lib" >> gpurun_out/r02qq/t.txt
  MPIX_LIB_PATH=$PWD/paper_2208_13707_b200/$lib timeout 300 python -m pytest tests/test_gpu_conventional.py -q --timeout 100 -p no:cacheprovider 2>&1 | tail -3 >> gpurun_out/r02qq/t.txt
done
