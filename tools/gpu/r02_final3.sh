# closing run on the final tree: whole GPU suite, smoke, the default bench line and its ncu launch list
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_suite.log 2>&1; echo "suite rc=$?"; tail -4 gpurun_out/r02_gpu_suite.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02_smoke.log
timeout 900 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-also > gpurun_out/r02_ncu_launch.log 2>&1; echo "launch rc=$?"
mkdir -p gpurun_out/table
python -c "
import json; d=json.load(open('gpurun_out/r02_bench_default.json')); print(d['ms_per_step'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['also']['c2-d3']['e2e'], d['also']['c2-d3']['ms_per_step'])"
for p in gram rownorms; do timeout 600 python bench.py --pass $p --config c5 --steps 3 --warmup 2 > gpurun_out/table/${p}_c5.json 2>/dev/null; done
python -c "
import json
for p in ('gram','rownorms'):
    d=json.load(open('gpurun_out/table/%s_c5.json'%p)); print(p, d['ms_per_step'], d['roofline']['frac'])"
