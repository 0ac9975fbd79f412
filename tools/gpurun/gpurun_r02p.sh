O=gpurun_out/r02p
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
ncu --set full --import-source on --clock-control none --cache-control none --warp-sampling-interval 0 -k regex:k_batch -s 20 -c 1 -o $O/kt8 python tools/profile_loopback.py --size 8 --steps 3 --warmup 20 > $O/ncu.log 2>&1
ncu -i $O/kt8.ncu-rep --page source --csv --print-source sass > $O/kt8_source_sass.csv 2>&1
ncu -i $O/kt8.ncu-rep --page details --csv > $O/kt8_details.csv 2>&1
rm -f $O/kt8.ncu-rep
