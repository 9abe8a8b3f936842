# which shared-memory configuration and time does each kernel get under the two libraries
O=gpurun_out/mode
mkdir -p $O
for lib in paper_2407_00656_b200/libhgks.so var/libhgks_divrcp.so; do
  tag=$(basename $lib .so)
  env HGKS_LIB=$PWD/$lib timeout 300 python bench.py --workload c2 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_$tag.json 2>&1
  python -c "
import json
d=json.loads(open('$O/bench_$tag.json').read().strip().splitlines()[-1])
print('live $tag', round(d['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if v['launches'] and v['avg_ms']>0.03})"
  env HGKS_LIB=$PWD/$lib timeout 300 ncu --clock-control none --cache-control none --metrics gpu__time_duration.sum,launch__shared_mem_config_size,launch__occupancy_limit_shared_mem,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct \
     -k regex:"k_flux|k_recon" -c 8 --csv --log-file $O/ncu_$tag.csv python bench.py --workload c2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  python - <<PY
import csv, collections
rows=[r for r in csv.reader(open('$O/ncu_$tag.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value')
for r in rows[1:]:
    pass
agg=collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    agg[r[ki][:34]][r[mi]].append(r[vi])
for k,m in agg.items():
    print('  ncu $tag', k, {mm: v[:4] for mm,v in m.items()})
PY
done
