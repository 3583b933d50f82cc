mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -k whole_trial > gpurun_out/r02_fullsize.log 2>&1; echo "fullsize rc=$?"; tail -4 gpurun_out/r02_fullsize.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "split or lattice or edge or empty" > gpurun_out/r02_split_tests.log 2>&1; echo "split tests rc=$?"; tail -2 gpurun_out/r02_split_tests.log
timeout 300 python bench.py --pass split --steps 5 --warmup 3 > gpurun_out/r02_c5_split.log 2>&1; echo "split rc=$?"; tail -1 gpurun_out/r02_c5_split.log | cut -c1-700
