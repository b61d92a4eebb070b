python __graft_entry__.py > gpurun_out/build.log 2>&1
rm -f gpurun_out/ncu2_*.ncu-rep
for c in grid256 c3 c5; do
ncu --set full --import-source on --clock-control none -k regex:k_struct_solve -c 1 -o gpurun_out/ncu2_solve_$c python tools/struct_one.py $c > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:k_struct_lambda2 -c 1 -o gpurun_out/ncu2_lambda2_grid256 python tools/struct_one.py grid256 --l2 > /dev/null 2>&1
for w in c1 c2; do
ncu --set full --import-source on --clock-control none -k regex:k_power_fused -c 1 -o gpurun_out/ncu2_fused_$w python bench.py --workload $w --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:k_mc -c 1 -o gpurun_out/ncu2_mc_grid python bench.py --path mc --workload grid --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_build_eq4 -c 1 -o gpurun_out/ncu2_eq4_c5 python bench.py --path eq4 --workload c5 --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/ncu2_*
