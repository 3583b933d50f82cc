# compute-sanitizer evidence for every device pass: memcheck, racecheck, synccheck
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --leak-check full --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/r02_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/r02_memcheck.log
timeout 1200 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/r02_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/r02_racecheck.log
timeout 900 $CS --tool synccheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/r02_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -4 gpurun_out/r02_synccheck.log
