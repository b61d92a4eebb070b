# Regenerates every bench line committed under profiles/r01/ (run via gpurun from the repo root).
set -u
O=gpurun_out
python __graft_entry__.py > $O/build.log 2>&1
run() { local name=$1; shift; timeout 900 python bench.py "$@" > $O/$name.json 2> $O/$name.err; echo "$name rc=$?"; }
# FP64 op counts and DRAM bytes of the ALU-bound kernels first (-> profiles/traffic.json, used below)
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active
for w in c5 c3; do ncu --metrics $M --clock-control none -k regex:k_build_eq4 -c 1 --csv python bench.py --path eq4 --workload $w --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_eq4_metrics_$w.csv 2>/dev/null; done
for w in c1 grid; do ncu --metrics $M --clock-control none -k regex:k_mc -c 1 --csv python bench.py --path mc --workload $w --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_mc_metrics_$w.csv 2>/dev/null; done
python tools/update_traffic.py > $O/traffic_update.log 2>&1; echo "traffic rc=$?"
run bench_c5                                        # default line (N=1): c5 fp64, dense path
for w in c1 c2 c3 c4; do run bench_$w --workload $w --no-cpu-baseline; done
run bench_c5_f32 --dtype f32 --no-cpu-baseline
run bench_c5_exp --mode exp --no-cpu-baseline
run bench_ref_c5 --impl reference --steps 1
for w in c5 c3 c4 grid; do run bench_struct_$w --path structured --workload $w; done
for w in grid c5 c1; do run bench_spec_$w --path spectral --workload $w; done
for w in c5 c4; do run bench_spec_dense_$w --path spectral_dense --workload $w; done
for w in c5 c3; do run bench_eq4_$w --path eq4 --workload $w; done
for w in c1 grid; do run bench_mc_$w --path mc --workload $w --steps 3 --warmup 1; done
# launch list of the default command (cold-cache, serialised: shares only)
SPLIDAR_EAGER=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_c5_eager.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo launches rc=$?
