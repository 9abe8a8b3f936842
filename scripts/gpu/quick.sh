python -m pytest tests -m gpu -x -q -k "not table10" > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
for w in c2 c3; do for p in 64 32; do python bench.py --steps 200 --warmup 10 --precision $p --workload $w --no-cpu-baseline > gpurun_out/bench_${w}_$p.json 2>&1; done; done
for f in gpurun_out/bench_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f',round(d['value']/1e6,1),round(d['ms_per_step'],4),{k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if v['launches'] and v['avg_ms']>0.03}, d['roofline'] and round(d['roofline']['frac'],3))"; done
