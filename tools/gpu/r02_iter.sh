mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/r02_fused_tests.log 2>&1; echo "fused rc=$?"; tail -4 gpurun_out/r02_fused_tests.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "split or lattice or edge or empty" > gpurun_out/r02_split_tests.log 2>&1; echo "split tests rc=$?"; tail -3 gpurun_out/r02_split_tests.log
timeout 300 python bench.py --config c5 --pass split --steps 5 --warmup 3 > gpurun_out/r02_c5_split.log 2>&1; echo "split rc=$?"; tail -1 gpurun_out/r02_c5_split.log | cut -c1-900
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-also > gpurun_out/r02_c5_fused.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r02_c5_fused.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel'], d['e2e']['ms_per_step'])"
