# round 2: cluster-fused kernel (kid_fused.cu) tests + c5 bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/r02_fused_tests.log 2>&1
echo "fused tests rc=$?"; tail -15 gpurun_out/r02_fused_tests.log
timeout 900 python -m pytest tests/ -m gpu -q -x --deselect tests/test_gpu_fused.py --deselect tests/test_gpu_fullsize.py > gpurun_out/r02_gpu_all.log 2>&1
echo "all gpu rc=$?"; tail -8 gpurun_out/r02_gpu_all.log
timeout 300 python bench.py --config c5 --pass split --steps 5 --warmup 3 > gpurun_out/r02_c5_split.log 2>&1
echo "split rc=$?"; tail -1 gpurun_out/r02_c5_split.log | cut -c1-1200
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_c5_fused.log 2>&1
echo "bench rc=$?"; tail -1 gpurun_out/r02_c5_fused.log | cut -c1-3000
