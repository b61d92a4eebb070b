mkdir -p gpurun_out/s2
timeout 900 python -m pytest tests -m gpu -x -q -k "build_plan or fused or one_shot or host or cache" > gpurun_out/s2/t.log 2>&1; tail -2 gpurun_out/s2/t.log
python tools/e2e_probe.py c1; python tools/e2e_probe.py c2
for w in c1 c2; do for i in 1 2; do timeout 600 python bench.py --workload $w --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/s2/bench_$w.$i.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/s2/bench_$w.$i.json')); print('$w', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), round(d['e2e']['value']/d['value'],3))"; done; done
