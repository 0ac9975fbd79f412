# flakiness hunt: the suite twice, the bench three times (final state)
O=gpurun_out/r02flaky
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
for i in 1 2; do
  timeout 1800 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider > $O/pytest$i.txt 2>&1; echo "rc=$?" >> $O/pytest$i.txt
done
for i in 1 2 3; do
  timeout 900 python bench.py > $O/bench$i.json 2> $O/bench$i.err; echo "rc=$?" >> $O/bench$i.err
done
