# mid / high skeleton ranks at m = 100 (c2-d3 eps sweep, c3-d5): k_gram (auto) vs the cluster kernels (k_fused_w for n <= 32)
mkdir -p gpurun_out
for cfg in c2-d3 c2-d3-e4 c2-d3-e6 c2-d3-e8 c2-d2 c1; do
for path in 0 1; do
timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --path $path > gpurun_out/mid_${cfg}_p$path.json 2> gpurun_out/mid_${cfg}_p$path.err || tail -2 gpurun_out/mid_${cfg}_p$path.err
python - <<PY
import json
try:
    d = json.load(open("gpurun_out/mid_${cfg}_p$path.json"))
    print("$cfg path=$path r=%d ms=%.4f kernel=%s kms=%.4f frac=%.3f" % (d["config"]["skeleton_rank"], d["ms_per_step"], d["roofline"]["kernel"], d["roofline"]["kernel_ms"], d["roofline"]["frac"]))
except Exception as e:
    print("$cfg path=$path failed", e)
PY
done
done
