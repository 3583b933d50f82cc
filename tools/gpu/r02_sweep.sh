mkdir -p gpurun_out
for cfg in "8 32" "8 48" "12 48" "12 96" "12 64"; do set -- $cfg
timeout 300 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-also --eval-warps $1 --chunk-cols $2 > gpurun_out/sw.log 2>&1
echo "c5 ew=$1 cw=$2: $(tail -1 gpurun_out/sw.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
done
for cfg in "8 32" "8 48" "8 64"; do set -- $cfg
timeout 300 python bench.py --config c4-d16 --steps 3 --warmup 3 --no-cpu-baseline --no-also --eval-warps $1 --chunk-cols $2 > gpurun_out/sw.log 2>&1
echo "c4 ew=$1 cw=$2: $(tail -1 gpurun_out/sw.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
done
