mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/san_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/san_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/san_synccheck.log
