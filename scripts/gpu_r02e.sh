#!/bin/bash
# round-2 pass E: parity suite, compute-sanitizer (memcheck, racecheck, synccheck) on small cases
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_tests.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/sanitize_memcheck.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck.txt
timeout 1200 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python scripts/sanitize_cases.py cfg1 cfg3-2^3-p3 cfg5-2^3-p3 cfg1-sc > gpurun_out/sanitize_racecheck.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck.txt
timeout 1200 $CS --tool synccheck --error-exitcode 9 python scripts/sanitize_cases.py cfg1 cfg4-2^3-p3 cfg5-2^3-p3 > gpurun_out/sanitize_synccheck.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitize_synccheck.txt
echo done
