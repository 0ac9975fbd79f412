# same-box A/B: libmpix_old.so (serial load_op) vs libmpix.so (warp-parallel load_op)
O=gpurun_out/r02kk
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
for i in 1 2; do
for lib in libmpix_old.so libmpix.so; do
  echo "== $lib" >> $O/ab.txt
  MPIX_LIB_PATH=$PWD/paper_2208_13707_b200/$lib timeout 120 python tools/pingpong_probe.py >> $O/ab.txt 2>&1
  MPIX_LIB_PATH=$PWD/paper_2208_13707_b200/$lib MPIX_FORCE_SYS=1 timeout 120 python tools/pingpong_probe.py >> $O/ab.txt 2>&1
  MPIX_LIB_PATH=$PWD/paper_2208_13707_b200/$lib timeout 120 python tools/graph_loopback.py >> $O/ab.txt 2>&1
done
done
