# A/B of the k_gram register split: fused pass (recon) and mode K (gram) per config
for i in 1 2; do
  for v in 72 88; do
    for c in c2-d3 c2-d2 c1 c3-d5; do
      r=$(KID_CUDA_SO=tools/libkernid_cuda_r$v.so timeout 200 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["roofline"]["kernel_ms"])')
      g=$(KID_CUDA_SO=tools/libkernid_cuda_r$v.so timeout 200 python bench.py --pass gram --config $c --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["roofline"]["kernel_ms"])')
      echo "E=$v $c recon=$r gram=$g"
    done
  done
done
