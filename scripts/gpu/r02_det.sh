# deterministic build (no --split-compile) vs two --split-compile draws: isolated kernel times + live steps
O=gpurun_out/det
mkdir -p $O
for lib in var/libhgks_det.so var/libhgks_splitdraw.so var/libhgks_split2.so; do
  tag=$(basename $lib .so)
  for w in c2 c5; do
    steps=200; [ $w = c5 ] && steps=40
    env HGKS_LIB=$PWD/$lib timeout 300 python bench.py --workload $w --steps $steps --warmup 5 --no-cpu-baseline > $O/bench_${w}_$tag.json 2>&1
    python -c "
import json
d=json.loads(open('$O/bench_${w}_$tag.json').read().strip().splitlines()[-1])
print('live $w $tag', '%.4g'%d['value'], round(d['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if v['launches'] and v['avg_ms']>0.03})"
  done
  env HGKS_LIB=$PWD/$lib timeout 300 ncu --clock-control none --cache-control none --metrics gpu__time_duration.sum \
     -k regex:"k_flux|k_recon" -c 8 --csv --log-file $O/ncu_$tag.csv python bench.py --workload c2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  python - <<PY
import csv, collections
rows=[r for r in csv.reader(open('$O/ncu_$tag.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(list)
for r in rows[1:]: agg[r[ki][:30]].append(float(r[vi].replace(',','')))
print('  ncu $tag', {k: round(sum(v)/len(v)/1e3,1) for k,v in agg.items()})
PY
done
