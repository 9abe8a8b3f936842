# moment-form flux with Newton reciprocals: isolated kernel times (ncu, two draws each) on C3
O=gpurun_out/mf
mkdir -p $O
HGKS_LIB=$PWD/var/libhgks_mf1a.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sphere or hex_box or walled or prandtl or dq0 or c1s" > $O/tests.log 2>&1; tail -1 $O/tests.log
for lib in var/libhgks_mf0a.so var/libhgks_mf0b.so var/libhgks_mf1a.so var/libhgks_mf1b.so; do
  tag=$(basename $lib .so)
  env HGKS_LIB=$PWD/$lib timeout 300 ncu --clock-control none --cache-control none --metrics gpu__time_duration.sum \
     -k regex:"k_flux" -c 6 --csv --log-file $O/ncu_$tag.csv python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  python - <<PY
import csv, collections
rows=[r for r in csv.reader(open('$O/ncu_$tag.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(list)
for r in rows[1:]: agg[r[ki][:30]].append(float(r[vi].replace(',','')))
print('ncu $tag', {k: round(sum(v)/len(v)/1e3,1) for k,v in agg.items()})
PY
done
