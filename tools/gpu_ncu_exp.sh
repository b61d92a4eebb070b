python __graft_entry__.py > gpurun_out/build.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
for dt in f64 f32; do for mode in exp factored; do
SPLIDAR_EAGER=1 ncu --metrics $M --clock-control none -k regex:k_build -c 1 --csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --dtype $dt --mode $mode > gpurun_out/ncu_build_${mode}_${dt}.csv 2> gpurun_out/ncu_build_${mode}_${dt}.err
done; done
for f in gpurun_out/ncu_build_*.csv; do echo $f; grep k_build $f | awk -F'","' '{print $13, $15}'; done
