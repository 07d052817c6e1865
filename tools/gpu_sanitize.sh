# compute-sanitizer over tools/sanitize_cases.py (every kernel of the library)
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 600 python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1; echo "exit=$?" >> gpurun_out/sanitize_plain.log
timeout 1500 $CS --tool memcheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "exit=$?" >> gpurun_out/sanitize_memcheck.log
timeout 1500 $CS --tool synccheck --print-limit 20 python tools/sanitize_cases.py --quick > gpurun_out/sanitize_synccheck.log 2>&1; echo "exit=$?" >> gpurun_out/sanitize_synccheck.log
timeout 2400 $CS --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_cases.py --quick > gpurun_out/sanitize_racecheck.log 2>&1; echo "exit=$?" >> gpurun_out/sanitize_racecheck.log
