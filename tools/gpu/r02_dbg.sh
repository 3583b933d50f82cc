mkdir -p gpurun_out
timeout 120 python tools/gpu/lev_debug.py > gpurun_out/lev_debug.log 2>&1; echo "lev rc=$?"; cat gpurun_out/lev_debug.log | tail -12
# ncu: the c5 fused pass (one step) -- launch list then a full capture of k_fused
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fused --csv --log-file gpurun_out/r02_c5_launches.csv python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-also > gpurun_out/r02_ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 1 -o gpurun_out/r02_k_fused_c5 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-also > gpurun_out/r02_ncu_full.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/r02_ncu_full.log
