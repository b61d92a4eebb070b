for d in . snapA; do (cd $d && python __graft_entry__.py > /dev/null 2>&1); done
for d in . snapA; do (cd $d && SPLIDAR_EAGER=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_power_step -c 40 --csv --log-file /tmp/l.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1; python -c "
import csv
rows=[r for r in csv.reader(open('/tmp/l.csv')) if len(r)>10]
h=rows[0]; vi=h.index('Metric Value')
v=[float(r[vi].replace(',','')) for r in rows[1:]]
print('$d', 'avg %.1f us over %d' % (sum(v)/len(v)/1e3, len(v)))"); done
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=400 2>&1 | tail -1
