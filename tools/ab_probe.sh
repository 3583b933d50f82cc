for i in 1 2 3; do
  for v in base ftz; do
    echo "== $v"; KID_CUDA_SO=tools/libkernid_cuda_$v.so PROBE_DBG=0 PROBE_TRACE= timeout 120 python tools/gram_probe.py c2-d3 2>&1 | grep "dbg=0"
  done
done
