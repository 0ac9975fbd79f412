# same-box A/B: every blocking receive polls (old) vs only receives <= an eager slot (new)
O=gpurun_out/r02pp
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
for i in 1 2; do
for lib in libmpix_old.so libmpix.so; do
  echo "== $lib" >> $O/ab.txt
  MPIX_LIB_PATH=$PWD/paper_2208_13707_b200/$lib timeout 120 python tools/pingpong_probe.py >> $O/ab.txt 2>&1
  MPIX_LIB_PATH=$PWD/paper_2208_13707_b200/$lib MPIX_FORCE_SYS=1 timeout 120 python tools/pingpong_probe.py >> $O/ab.txt 2>&1
done
done
timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_ll.py tests/test_gpu_model_check.py tests/test_gpu_staging.py tests/test_gpu_batch.py tests/test_gpu_conventional.py tests/test_gpu_graph.py tests/test_gpu_paths.py -q -x --timeout 200 -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
