# out-of-bounds evidence for every device pass without compute-sanitizer: the -DKID_GUARD library
mkdir -p gpurun_out
python paper_1409_2802_b200/build.py --guard > gpurun_out/r02_guard_build.log 2>&1; echo "guard build rc=$?"
timeout 1500 python tools/guard_cases.py > gpurun_out/r02_guard_cases.log 2>&1; echo "guard rc=$?"; tail -6 gpurun_out/r02_guard_cases.log
