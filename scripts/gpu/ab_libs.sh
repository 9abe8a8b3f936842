# A/B of alternative library builds: bash scripts/gpu/ab_libs.sh "lib1 lib2 ..." [bench args]
LIBS=$1; shift
for lib in $LIBS; do
  tag=$(basename $lib .so)
  timeout 180 env HGKS_LIB=$PWD/$lib python bench.py --steps 300 --warmup 10 --no-cpu-baseline "$@" > gpurun_out/abl_$tag.json 2>&1
  python -c "
import json
try:
  d=json.loads(open('gpurun_out/abl_$tag.json').read().strip().splitlines()[-1])
  print('$tag $*', round(d['value']/1e6,1), round(d['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if v['launches'] and v['avg_ms']>0.03})
except Exception as e: print('$tag FAILED', open('gpurun_out/abl_$tag.json').read()[-300:])"
done
