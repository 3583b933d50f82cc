# refresh of the closing evidence after k_gram2: default bench line, its ncu launch list, ncu --set full of k_gram2
# at c5, the Gram rows of the table; then the whole GPU suite
mkdir -p gpurun_out gpurun_out/table
timeout 900 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-also > gpurun_out/r02_ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_gram2 -c 1 -f -o gpurun_out/r02_k_gram2_c5 python bench.py --pass gram --config c5 --steps 1 --warmup 1 > gpurun_out/r02_ncu_g2c5.log 2>&1; echo "ncu g2 rc=$?"
python tools/ncu_brief.py gpurun_out/r02_k_gram2_c5.ncu-rep > gpurun_out/r02_k_gram2_c5.txt 2>&1
for c in c2-d3 c4-d16 c5; do
  timeout 600 python bench.py --pass gram --config $c --steps 5 --warmup 3 > gpurun_out/table/gram_$c.json 2>/dev/null
done
for c in c4-d16 c5; do
  timeout 600 python bench.py --pass leverage --config $c --steps 3 --warmup 2 > gpurun_out/table/leverage_$c.json 2>/dev/null
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/table/*.json")):
    try:
        d = json.load(open(f))
        r = d.get("roofline", {})
        print(f.split("/")[-1][:-5], "ms=%.4f" % d["ms_per_step"], "value=%.4g" % d["value"], d["unit"], "kernel=%s" % r.get("kernel"), "frac=%.3f" % r.get("frac", float("nan")))
    except Exception as e:
        print(f, "failed", e)
PY
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_suite.log 2>&1; echo "suite rc=$?"; tail -4 gpurun_out/r02_gpu_suite.log
