mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/r02_fused_tests.log 2>&1; echo "fused rc=$?"; tail -3 gpurun_out/r02_fused_tests.log
for ew in 8 12; do
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-also --eval-warps $ew > gpurun_out/r02_c5_ew$ew.log 2>&1; echo "c5 ew=$ew rc=$?"; tail -1 gpurun_out/r02_c5_ew$ew.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel'])"
done
timeout 600 python bench.py --config c4-d16 --steps 5 --warmup 3 --no-cpu-baseline --no-also > gpurun_out/r02_c4.log 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/r02_c4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel'], d['config']['skeleton_rank'], d['e2e']['ms_per_step'])"
