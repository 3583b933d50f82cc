# the warp-tile kernel, one CTA per SM (solo) vs the CTA pair: parity tests, then c5 and the mid-rank shapes
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py tests/test_gpu_mirror.py tests/test_gpu_svd.py -x -q > gpurun_out/solo_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/solo_tests.log
run() {
timeout 600 python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline --no-also --tile-form $3 --tile-warps $4 > gpurun_out/solo_$1_f$3_w$4.json 2> gpurun_out/solo_$1_f$3_w$4.err || tail -2 gpurun_out/solo_$1_f$3_w$4.err
python - <<PY
import json
try:
    d = json.load(open("gpurun_out/solo_$1_f$3_w$4.json"))
    print("$1 form=$3 warps=$4 r=%d ms=%.4f kernel=%s kms=%.4f frac=%.3f" % (d["config"]["skeleton_rank"], d["ms_per_step"], d["roofline"]["kernel"], d["roofline"]["kernel_ms"], d["roofline"]["frac"]))
except Exception as e:
    print("$1 form=$3 warps=$4 failed", e)
PY
}
run c5 5 1 0
run c5 5 2 8
run c2-d3-e6 20 1 0
run c2-d3-e6 20 1 8
run c2-d3-e6 20 2 0
run c5 5 2 0
run c2-d3 20 0 0
run c3-d5 20 0 0
run c4-d16-e8 5 0 0
run c5-e8 5 0 0
