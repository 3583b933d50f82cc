# Round summary: every pass x config through bench.py (one JSON line each) -> gpurun_out/table/
mkdir -p gpurun_out/table
for c in c1 c2-d2 c2-d3 c3-d5 c4-d16 c5-d8-shard; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/table/recon_$c.json 2>/dev/null
  for p in gram leverage svd rownorms split; do
    timeout 300 python bench.py --pass $p --config $c --steps 5 --warmup 3 > gpurun_out/table/${p}_$c.json 2>/dev/null
  done
done
for c in c1 c2-d3 c3-d5; do
  timeout 300 python bench.py --pass tsqr --config $c --steps 5 --warmup 3 > gpurun_out/table/tsqr_$c.json 2>/dev/null
  timeout 300 python bench.py --pass apply --config $c --steps 10 --warmup 3 > gpurun_out/table/apply_$c.json 2>/dev/null
done
