mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-also > gpurun_out/r02_ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_w -c 1 -o gpurun_out/r02_k_fused_w_c5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-also > gpurun_out/r02_ncu_fw.log 2>&1; echo "ncu fw rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:"k_dist_flag|k_compact_flag" -c 2 -o gpurun_out/r02_split_c5 python bench.py --pass split --steps 1 --warmup 3 > gpurun_out/r02_ncu_split.log 2>&1; echo "ncu split rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 1 -o gpurun_out/r02_k_fused_c4 python bench.py --config c4-d16 --steps 1 --warmup 3 --no-cpu-baseline --no-also > gpurun_out/r02_ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
