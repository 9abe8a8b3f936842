# A/B of an environment switch on the bench: bash scripts/gpu/ab_env.sh VAR "v1 v2" [bench args]
VAR=$1; VALS=$2; shift 2
for v in $VALS; do
  env $VAR=$v python bench.py --steps 200 --warmup 10 --no-cpu-baseline "$@" > gpurun_out/ab_$v.json 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1])
print('$VAR=$v $*',round(d['value']/1e6,1),round(d['ms_per_step'],4),{k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if v['launches'] and v['avg_ms']>0.03})"
done
