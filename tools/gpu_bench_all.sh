# Regenerates every bench line committed under profiles/r02/ (run via gpurun from the repo root).
set -u
O=gpurun_out
mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
run() { local name=$1; shift; timeout 900 python bench.py "$@" > $O/$name.json 2> $O/$name.err; echo "$name rc=$?"; }
run bench_c5 --steps 20 --warmup 5                   # default line (N=1): c5 fp64, dense path
for w in c1 c2 c3 c4; do run bench_$w --workload $w --no-cpu-baseline --steps 20 --warmup 5; done
run bench_c5_f32 --dtype f32 --no-cpu-baseline --steps 20 --warmup 5
run bench_c5_exp --mode exp --no-cpu-baseline
run bench_c5_rows --shard rows --no-cpu-baseline
run bench_ref_c5 --impl reference --steps 1
for w in c5 c3 c4 grid; do run bench_struct_$w --path structured --workload $w; done
for w in grid c5 c1; do run bench_spec_$w --path spectral --workload $w; done
for w in c5 c4; do run bench_spec_dense_$w --path spectral_dense --workload $w; done
for w in c5 c3; do run bench_eq4_$w --path eq4 --workload $w; done
for w in c1 grid; do run bench_mc_$w --path mc --workload $w --steps 3 --warmup 1; done
# launch lists of the default and fp32 commands (eager: ncu does not descend into conditional graph
# bodies), each after the same command exited 0 above; then one NVTX-filtered list (only the kernels
# launched inside splidar_plan_launch calls)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5_f64.csv \
    env SPLIDAR_EAGER=1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_f64.log 2>&1; echo "ncu f64 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5_f32.csv \
    env SPLIDAR_EAGER=1 python bench.py --steps 2 --warmup 3 --dtype f32 --no-cpu-baseline > $O/ncu_f32.log 2>&1; echo "ncu f32 rc=$?"
ncu --nvtx --nvtx-include "splidar_plan_launch/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_nvtx_c4.csv env SPLIDAR_EAGER=1 python bench.py --workload c4 --steps 1 --warmup 3 \
    --no-cpu-baseline > $O/ncu_nvtx.log 2>&1; echo "ncu nvtx rc=$?"
