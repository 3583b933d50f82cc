# round 2: cluster-fused kernel (kid_fused.cu) tests + c5 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/r02_fused_tests.log 2>&1
echo "fused tests rc=$?"; tail -15 gpurun_out/r02_fused_tests.log
timeout 900 python -m pytest tests/ -m gpu -q -x --deselect tests/test_gpu_fused.py > gpurun_out/r02_gpu_all.log 2>&1
echo "all gpu rc=$?"; tail -8 gpurun_out/r02_gpu_all.log
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_c5_fused.log 2>&1
echo "bench rc=$?"; tail -2 gpurun_out/r02_c5_fused.log | cut -c1-900
