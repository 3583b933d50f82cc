# randomised differential check of the Gram-type passes across kernel families (tools/fuzz_kernels.py)
mkdir -p gpurun_out
timeout 2400 python tools/fuzz_kernels.py 800 11 > gpurun_out/r02_fuzz.log 2>&1; echo "fuzz rc=$?"; tail -12 gpurun_out/r02_fuzz.log
