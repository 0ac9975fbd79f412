# same-box A/B of the host path: libmpix_old.so vs libmpix.so, cfg4 message rate
O=gpurun_out/r02mm
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
for i in 1 2; do
for lib in libmpix_old.so libmpix.so; do
  echo "== $lib" >> $O/ab.txt
  MPIX_LIB_PATH=$PWD/paper_2208_13707_b200/$lib timeout 300 python tools/scratch/msgrate_probe.py >> $O/ab.txt 2>&1
done
done
timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_batch.py tests/test_gpu_conventional.py tests/test_gpu_staging.py tests/test_gpu_graph.py -q -x --timeout 200 -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
