# the three-phase residual kernel k_resid3 against k_gram (KID_OPT_KERNEL 4): parity tests, fuzz, then the m = 100 configs
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mirror.py tests/test_gpu_svd.py -x -q > gpurun_out/resid3_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/resid3_tests.log
timeout 600 python tools/fuzz_kernels.py 300 3 > gpurun_out/resid3_fuzz.log 2>&1; echo "fuzz rc=$?"; tail -3 gpurun_out/resid3_fuzz.log
for cfg in c2-d3 c2-d2 c2-d3-e4 c1; do
for k in 0 4; do
timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --kernel $k > gpurun_out/resid3_${cfg}_k$k.json 2> gpurun_out/resid3_${cfg}_k$k.err || tail -2 gpurun_out/resid3_${cfg}_k$k.err
python - <<PY
import json
try:
    d = json.load(open("gpurun_out/resid3_${cfg}_k$k.json"))
    print("$cfg kernel-opt=$k r=%d ms=%.4f kernel=%s kms=%.4f frac=%.3f" % (d["config"]["skeleton_rank"], d["ms_per_step"], d["roofline"]["kernel"], d["roofline"]["kernel_ms"], d["roofline"]["frac"]))
except Exception as e:
    print("$cfg k=$k failed", e)
PY
done
done
