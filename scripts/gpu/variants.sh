# A/B of alternative builds on the c2 bench: bash scripts/gpu/variants.sh lib1.so lib2.so ...
for lib in "$@"; do
  HGKS_LIB=$PWD/$lib python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/var_$(basename $lib .so).json 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/var_$(basename $lib .so).json').read().strip().splitlines()[-1])
print('$lib',round(d['value']/1e6,1),round(d['ms_per_step'],4),{k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if v['launches'] and v['avg_ms']>0.03})"
done
