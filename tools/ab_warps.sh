# A/B of the k_gram eval / MMA warp split (tools/libkernid_cuda_w<EW>.so built with kEW = EW)
for i in 1 2; do
  for v in 12 13 14; do
    for c in c2-d3 c2-d2 c3-d5; do
      r=$(KID_CUDA_SO=tools/libkernid_cuda_w$v.so timeout 200 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["roofline"]["kernel_ms"])')
      g=$(KID_CUDA_SO=tools/libkernid_cuda_w$v.so timeout 200 python bench.py --pass gram --config $c --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["roofline"]["kernel_ms"])')
      echo "EW=$v $c recon=$r gram=$g"
    done
  done
done
