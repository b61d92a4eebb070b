python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_eq4_gpu.py -m gpu -q --timeout=240 > gpurun_out/pytest_eq4.log 2>&1; tail -2 gpurun_out/pytest_eq4.log
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active
for w in c5 c3; do
ncu --metrics $M --clock-control none -k regex:k_build_eq4 -c 1 --csv python bench.py --path eq4 --workload $w --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_eq4_metrics_$w.csv 2>gpurun_out/ncu_eq4_metrics_$w.err
done
grep -h k_build_eq4 gpurun_out/ncu_eq4_metrics_*.csv | cut -c1-300
