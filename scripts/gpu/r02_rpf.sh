# flux record prefetch-ahead variants vs the default build, C2 and C5, two rounds
O=gpurun_out/rpf
mkdir -p $O
for round in 1 2; do
for w in c2 c5; do
  steps=300; [ $w = c5 ] && steps=60
  for lib in paper_2407_00656_b200/libhgks.so var/libhgks_rpf32.so var/libhgks_rpf128.so; do
    tag=$(basename $lib .so)
    timeout 300 env HGKS_LIB=$PWD/$lib python bench.py --steps $steps --warmup 5 --workload $w --no-cpu-baseline > $O/bench_${w}_${tag}_$round.json 2>&1
    python -c "
import json
d=json.loads(open('$O/bench_${w}_${tag}_$round.json').read().strip().splitlines()[-1])
print('$w $tag $round', '%.4g'%d['value'], round(d['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if v['launches'] and v['avg_ms']>0.03})"
  done
done
done
