O=gpurun_out/r02j
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:k_batch -s 5 -c 1 -o $O/kb8 python tools/profile_loopback.py --size 8 --steps 3 --warmup 5 > $O/ncu.log 2>&1
ncu -i $O/kb8.ncu-rep --page source --csv --print-source sass > $O/kb8_source_sass.csv 2>&1
ncu -i $O/kb8.ncu-rep --page source --csv --print-source cuda > $O/kb8_source_cuda.csv 2>&1
ncu -i $O/kb8.ncu-rep --page raw --csv > $O/kb8_raw.csv 2>&1
ncu -i $O/kb8.ncu-rep --page details --csv > $O/kb8_details.csv 2>&1
rm -f $O/kb8.ncu-rep
