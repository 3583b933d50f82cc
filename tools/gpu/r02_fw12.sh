# A/B of the warp-tile kernel at 8 vs 12 warps per CTA (c5), after the parity tests of the cluster kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_fullsize.py -x -q > gpurun_out/fw12_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/fw12_tests.log
for w in 8 12; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-also --tile-warps $w > gpurun_out/fw12_bench_w$w.json 2> gpurun_out/fw12_bench_w$w.err; echo "bench w=$w rc=$?"
python - <<PY
import json
d = json.load(open("gpurun_out/fw12_bench_w$w.json"))
print("w=$w", d["ms_per_step"], d["roofline"]["kernel"], d["roofline"]["kernel_ms"], d["roofline"]["frac"])
PY
done
