# dense lambda_2: timing lines + the eager-mode launch list (kernel shares) at config 5
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 300 python tools/spec_dense_time.py > gpurun_out/spec_dense_time.jsonl 2>&1; cat gpurun_out/spec_dense_time.jsonl
SPLIDAR_EAGER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_spec_dense_c5.csv python tools/sd_one.py > gpurun_out/ncu_sd.log 2>&1; tail -2 gpurun_out/ncu_sd.log
