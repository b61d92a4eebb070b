for c in grid256 c3 c5; do
ncu --set full --import-source on --clock-control none -k regex:k_struct_solve -c 1 -o gpurun_out/ncu_struct_$c python tools/struct_one.py $c > gpurun_out/ncu_struct_$c.log 2>&1
done
ls -la gpurun_out
