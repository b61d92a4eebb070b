python __graft_entry__.py > gpurun_out/build.log 2>&1
python __graft_entry__.py --smoke 2>&1 | tail -1 | cut -c1-120
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=400 > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for w in c5 c4 c3; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -c 300 gpurun_out/bench_$w.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); r=d['roofline']; print('$w', round(d['value'],1), round(d['ms_per_step'],3), round(d['ms_solve_per_step'],3), round(r['frac'],3), d['iterations'][0][:6])"; done
# check-kernel time per launch from the eager launch list of the default step
SPLIDAR_EAGER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_c5_eager.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ncu_c5.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/launches_c5_eager.csv")) if len(r) > 5]
h = rows[0]; ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    v = float(r[vi].replace(",", "")) * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r[ui], 1.0)
    agg[r[ki].split("(")[0]][0] += 1; agg[r[ki].split("(")[0]][1] += v
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:5]:
    print(f"{k[:50]:50s} {n:4d} {v / n:9.1f} us/launch")
PY
