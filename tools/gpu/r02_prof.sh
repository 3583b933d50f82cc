mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 1 -o gpurun_out/r02_k_fused_c5_v3 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-also --eval-warps 12 --chunk-cols 64 > gpurun_out/r02_ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 1 -o gpurun_out/r02_k_fused_c4_v1 python bench.py --config c4-d16 --steps 1 --warmup 3 --no-cpu-baseline --no-also --chunk-cols 48 > gpurun_out/r02_ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
