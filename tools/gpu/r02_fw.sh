mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/r02_fused_tests.log 2>&1; echo "fused rc=$?"; tail -4 gpurun_out/r02_fused_tests.log
for k in 2 1; do
timeout 300 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-also --kernel $k --eval-warps 12 --chunk-cols 64 > gpurun_out/sw.log 2>&1
echo "c5 kernel=$k: $(tail -1 gpurun_out/sw.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), round(d['roofline']['frac'],3), d['roofline']['kernel'])" 2>&1 | tail -1)"
done
