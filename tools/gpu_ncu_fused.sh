python __graft_entry__.py > gpurun_out/build.log 2>&1
for w in c1 c2; do
ncu --set full --import-source on --clock-control none -k regex:k_power_fused -c 1 -o gpurun_out/ncu_fused_$w python bench.py --workload $w --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_fused_$w.log 2>&1
done
ls gpurun_out/*.ncu-rep
