# ncu --set full captures of the kernels added / reworked late in r01, and the structured bench lines
python __graft_entry__.py > gpurun_out/build.log 2>&1
rm -f gpurun_out/ncu3_*.ncu-rep
for c in c4 c5; do
ncu --set full --import-source on --clock-control none -k regex:k_struct_solve_c1 -c 1 -o gpurun_out/ncu3_solve_c1_$c python tools/struct_one.py $c > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:k_struct_lambda2 -c 1 -o gpurun_out/ncu3_lambda2_c5 python tools/struct_one.py c5 --l2 > /dev/null 2>&1
SPLIDAR_EAGER=1 ncu --set full --import-source on --clock-control none -k regex:"k_sd_dots|k_power_step" -s 30 -c 2 -o gpurun_out/ncu3_sd_c5 python tools/sd_one.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_vec_a -c 1 -o gpurun_out/ncu3_vec_a_c5 python tools/struct_one.py c5 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_vec_small -c 1 -o gpurun_out/ncu3_vec_small_c3 python tools/struct_one.py c3 > /dev/null 2>&1
SPLIDAR_EAGER=1 ncu --set full --import-source on --clock-control none -k regex:k_power_check -s 5 -c 1 -o gpurun_out/ncu3_check_c5 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
ls gpurun_out/ncu3_*
run() { local name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/$name.json 2> gpurun_out/$name.err; echo "$name rc=$?"; }
for w in c5 c3 c4 grid; do run bench_struct_$w --path structured --workload $w; done
for w in grid c5 c1; do run bench_spec_$w --path spectral --workload $w; done
