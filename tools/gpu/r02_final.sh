# round-2 closing evidence: whole GPU suite, the default bench line, its ncu launch list, ncu --set full of the
# headline kernel (k_fused_w, one CTA per SM, c5) and of the mid-rank shape, the per-config table
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_suite.log 2>&1; echo "suite rc=$?"; tail -4 gpurun_out/r02_gpu_suite.log
timeout 900 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-also > gpurun_out/r02_ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_w -c 1 -f -o gpurun_out/r02_k_fused_w_solo_c5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-also > gpurun_out/r02_ncu_fw.log 2>&1; echo "ncu fw rc=$?"
python tools/ncu_brief.py gpurun_out/r02_k_fused_w_solo_c5.ncu-rep > gpurun_out/r02_k_fused_w_solo_c5.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused_w -c 1 -f -o gpurun_out/r02_k_fused_w_solo_c2d3e6 python bench.py --config c2-d3-e6 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_fw2.log 2>&1; echo "ncu fw2 rc=$?"
python tools/ncu_brief.py gpurun_out/r02_k_fused_w_solo_c2d3e6.ncu-rep > gpurun_out/r02_k_fused_w_solo_c2d3e6.txt 2>&1
mkdir -p gpurun_out/table
for c in c1 c2-d2 c2-d3 c2-d3-e4 c2-d3-e6 c2-d3-e8 c3-d5 c4-d16 c4-d16-e8 c4-d64-unfiltered c5-e8; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/table/recon_$c.json 2>/dev/null
done
for c in c2-d3 c4-d16 c5; do
  for p in split gram; do
    timeout 600 python bench.py --pass $p --config $c --steps 5 --warmup 3 > gpurun_out/table/${p}_$c.json 2>/dev/null
  done
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
