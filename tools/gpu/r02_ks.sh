mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/r02_fused_tests.log 2>&1; echo "fused rc=$?"; tail -3 gpurun_out/r02_fused_tests.log
for cfg in "12 64" "12 96" "12 32"; do set -- $cfg
timeout 300 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-also --eval-warps $1 --chunk-cols $2 > gpurun_out/sw.log 2>&1
echo "c5 ew=$1 cw=$2: $(tail -1 gpurun_out/sw.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
done
