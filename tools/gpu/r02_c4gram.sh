mkdir -p gpurun_out
timeout 600 python bench.py --config c4-d16 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_c4.log 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/r02_c4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel'], d['config']['skeleton_rank'], d['e2e']['ms_per_step'])"
timeout 600 python bench.py --config c5 --pass gram --steps 2 --warmup 3 > gpurun_out/r02_c5_gram.log 2>&1; echo "gram rc=$?"; tail -1 gpurun_out/r02_c5_gram.log | cut -c1-700
timeout 600 python bench.py --config c4-d16 --pass gram --steps 3 --warmup 3 > gpurun_out/r02_c4_gram.log 2>&1; echo "c4 gram rc=$?"; tail -1 gpurun_out/r02_c4_gram.log | cut -c1-700
