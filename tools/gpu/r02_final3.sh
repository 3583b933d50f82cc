# closing run on the final tree: whole GPU suite, smoke, the default bench line and its ncu launch list
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_suite.log 2>&1; echo "suite rc=$?"; tail -4 gpurun_out/r02_gpu_suite.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02_smoke.log
timeout 900 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-also > gpurun_out/r02_ncu_launch.log 2>&1; echo "launch rc=$?"
mkdir -p gpurun_out/table
python -c "
import json; d=json.load(open('gpurun_out/r02_bench_default.json')); print(d['ms_per_step'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['also']['c2-d3']['e2e'], d['also']['c2-d3']['ms_per_step'])"
timeout 900 ncu --set full --clock-control none -k regex:"k_dist_flag|k_compact_flag|k_split_rank" -c 3 -f -o gpurun_out/r02_split_c5_final python bench.py --pass split --steps 1 --warmup 3 > gpurun_out/r02_ncu_split.log 2>&1; echo "ncu split rc=$?"
ncu -i gpurun_out/r02_split_c5_final.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv, sys
rows = list(csv.reader(sys.stdin))
h = rows[0]
keys = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']
idx = [h.index(k) for k in keys if k in h]
print(', '.join(h[i] for i in idx)); print(', '.join(rows[1][i] for i in idx))
for r in rows[2:]: print(', '.join(r[i] for i in idx))
" > gpurun_out/r02_split_c5_final.txt 2>&1
