# memcheck then racecheck of a small end-to-end workload (after a plain run)
python tools/sanitize_target.py > gpurun_out/san_plain.log 2>&1 || exit 1
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 3 --print-limit 50 python tools/sanitize_target.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck.log
