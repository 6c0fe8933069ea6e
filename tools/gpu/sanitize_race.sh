python tools/sanitize_target.py > gpurun_out/san_plain2.log 2>&1 || exit 1
timeout 3000 compute-sanitizer --tool racecheck --racecheck-report all --error-exitcode 3 --print-limit 50 python tools/sanitize_target.py > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/san_racecheck.log
