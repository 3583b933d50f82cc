mkdir -p gpurun_out
./tools/fp64_peaks > gpurun_out/r02_fp64_peaks.log 2>&1; echo "peaks rc=$?"; grep sustained gpurun_out/r02_fp64_peaks.log
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/r02_fused_tests.log 2>&1; echo "fused rc=$?"; tail -2 gpurun_out/r02_fused_tests.log
timeout 900 python bench.py > gpurun_out/r02_bench_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r02_bench_default.log
timeout 600 python bench.py --config c4-d16 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_c4.log 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/r02_c4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel'], d['config']['skeleton_rank'], d['e2e']['ms_per_step'])"
