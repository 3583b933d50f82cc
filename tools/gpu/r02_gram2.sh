# the two-phase Gram kernel k_gram2 against the cluster kernel k_fused (Gram mode): parity tests, then c4 / c5
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fused.py tests/test_gpu_spectrum.py -x -q > gpurun_out/gram2_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gram2_tests.log
for cfg in c4-d16 c5; do
for k in 0; do
timeout 600 python bench.py --pass gram --config $cfg --steps 3 --warmup 2 --kernel $k > gpurun_out/gram2_${cfg}_k$k.json 2> gpurun_out/gram2_${cfg}_k$k.err || tail -2 gpurun_out/gram2_${cfg}_k$k.err
python - <<PY
import json
try:
    d = json.load(open("gpurun_out/gram2_${cfg}_k$k.json"))
    print("$cfg kernel-opt=$k ms=%.3f kernel=%s kms=%.3f frac=%.3f" % (d["ms_per_step"], d["roofline"]["kernel"], d["roofline"]["kernel_ms"], d["roofline"]["frac"]))
except Exception as e:
    print("$cfg k=$k failed", e)
PY
done
done
