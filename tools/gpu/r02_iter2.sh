mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/r02_fused_tests.log 2>&1; echo "fused rc=$?"; tail -4 gpurun_out/r02_fused_tests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 1 -o gpurun_out/r02_k_fused_c5_v2 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-also > gpurun_out/r02_ncu_full.log 2>&1; echo "ncu full rc=$?"
