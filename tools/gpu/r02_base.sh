# round-2 baseline: c5 at N=1 through the current code
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out
( time python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline ) > gpurun_out/r02_c5_base.log 2>&1
tail -3 gpurun_out/r02_c5_base.log
