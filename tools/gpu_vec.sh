python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for w in c5 c4; do timeout 300 python bench.py --path structured --workload $w --no-cpu-baseline > gpurun_out/bench_struct_$w.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_struct_$w.json')); r=d['roofline']; print('$w', round(d['value']), round(d['ms_per_step'],4), round(r.get('kernel_ms_per_step'),4))"; done
SPLIDAR_EAGER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_vec --csv --log-file gpurun_out/vec.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/vec.csv")) if len(r) > 5]
h = rows[0]; ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
for r in rows[1:8]: print(r[ki][:40], r[vi], r[ui])
PY
