# ncu --set full of k_power_check (c5 fp64 and fp32 eager), after the same command exited 0 without ncu.
mkdir -p gpurun_out
python -m paper_2509_20500_b200.build > /dev/null
export SPLIDAR_EAGER=1
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/chk_plain.json 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_power_check" -s 20 -c 1 -o gpurun_out/chk_f64 \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/chk_ncu64.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_power_check" -s 20 -c 1 -o gpurun_out/chk_f32 \
    python bench.py --steps 1 --warmup 1 --dtype f32 --no-cpu-baseline --no-e2e > gpurun_out/chk_ncu32.log 2>&1
ls -la gpurun_out/chk_*
