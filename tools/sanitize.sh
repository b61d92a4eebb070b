#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py: memcheck, synccheck, initcheck, racecheck
# (graph path and eager path). Logs in gpurun_out/sanitize_*.log
mkdir -p gpurun_out
python -m paper_2509_20500_b200.build > /dev/null
python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/sanitize_plain.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck racecheck; do
  for eager in 0 1; do
    SPLIDAR_EAGER=$eager timeout 1500 $CS --tool $tool --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_cases.py > gpurun_out/sanitize_${tool}_eager${eager}.log 2>&1
    echo "rc=$?" >> gpurun_out/sanitize_${tool}_eager${eager}.log
    echo "$tool eager=$eager: $(grep -E 'ERROR SUMMARY|rc=' gpurun_out/sanitize_${tool}_eager${eager}.log | tr '\n' ' ')"
  done
done
