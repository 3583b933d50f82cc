mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r02_multi.log 2>&1; echo "multi rc=$?"; tail -3 gpurun_out/r02_multi.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_suite.log 2>&1; echo "suite rc=$?"; tail -8 gpurun_out/r02_gpu_suite.log
