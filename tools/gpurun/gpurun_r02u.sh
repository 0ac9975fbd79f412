O=gpurun_out/r02u
mkdir -p $O
export CUDA_MODULE_LOADING=EAGER
timeout 120 tools/stencil_probe 512 10 > $O/stencil_probe.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider --durations=30 > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
