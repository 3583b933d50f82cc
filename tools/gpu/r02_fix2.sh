mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q > gpurun_out/r02_fullsize.log 2>&1; echo "fullsize rc=$?"; tail -4 gpurun_out/r02_fullsize.log
bash tools/gpu/r02_sanitize.sh
