#!/bin/bash
# End-of-round evidence on one box (run via gpurun): full GPU suite, smoke, every bench line and the
# launch lists (tools/gpu_bench_all.sh), the fused solver's ncu captures (tools/gpu_fused_prof.sh).
mkdir -p gpurun_out
python -m paper_2509_20500_b200.build > /dev/null
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
tail -2 gpurun_out/gputest.log
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -1 gpurun_out/smoke.log
bash tools/gpu_bench_all.sh
bash tools/gpu_fused_prof.sh
