# round 2: first GPU run of the cluster-fused kernel (kid_fused.cu)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q > gpurun_out/r02_fused_tests.log 2>&1
echo "fused tests rc=$?"; tail -15 gpurun_out/r02_fused_tests.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_svd.py -x -q > gpurun_out/r02_parity.log 2>&1
echo "parity rc=$?"; tail -5 gpurun_out/r02_parity.log
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_c5_fused.log 2>&1
echo "bench rc=$?"; tail -2 gpurun_out/r02_c5_fused.log | cut -c1-1500
