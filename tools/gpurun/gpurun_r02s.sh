# N>1 launch paths on the 1-GPU box (--share-gpus validation, not measurements)
O=gpurun_out/r02s2
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500+N)) \
    bench.py --gpus $N --steps 5 --warmup 3 --share-gpus > $O/bench_n$N.json 2> $O/bench_n$N.err; echo "rc=$?" >> $O/bench_n$N.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 \
  bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $O/bench_ref_n2.json 2> $O/bench_ref_n2.err; echo "rc=$?" >> $O/bench_ref_n2.err
