python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_mc_gpu.py -m gpu -q --timeout=240 > gpurun_out/pytest_mc.log 2>&1; tail -3 gpurun_out/pytest_mc.log
for w in c1 grid; do timeout 600 python bench.py --path mc --workload $w --steps 3 --warmup 1 > gpurun_out/bench_mc_$w.json 2> gpurun_out/bench_mc_$w.err; tail -c 300 gpurun_out/bench_mc_$w.err; python -c "
import json; d=json.load(open('gpurun_out/bench_mc_$w.json')); print('$w', d['value'], d['ms_per_step'], d['registrations_per_step'], d['cpu_baseline'])"; done
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for w in c1 grid; do
ncu --metrics $M --clock-control none -k regex:k_mc -c 1 --csv python bench.py --path mc --workload $w --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_mc_metrics_$w.csv 2>gpurun_out/ncu_mc_metrics_$w.err
done
grep -h k_mc gpurun_out/ncu_mc_metrics_*.csv | awk -F'","' '{print $13, $15}'
grep -h registrations_per_step gpurun_out/ncu_mc_metrics_*.csv | python -c "
import sys,json
for l in sys.stdin:
    l=l[l.index('{'):]; d=json.loads(l); print(d['config']['workload'][:10], d['registrations_per_step'])"
