O=gpurun_out/r02dd
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
python tools/profile_selfsend.py 8 20 > $O/plain.txt 2>&1
ncu --set full --import-source on --clock-control none --cache-control none --warp-sampling-interval 0 -k regex:k_batch -s 10 -c 2 -o $O/ss python tools/profile_selfsend.py 8 20 > $O/ncu.log 2>&1
ncu -i $O/ss.ncu-rep --page source --csv --print-source sass > $O/ss_source_sass.csv 2>&1
ncu -i $O/ss.ncu-rep --page details --csv > $O/ss_details.csv 2>&1
rm -f $O/ss.ncu-rep
