# per-kernel durations + chosen smem config of library variants under identical (ncu) conditions, and live bench
O=gpurun_out/ab1
mkdir -p $O
for lib in paper_2407_00656_b200/libhgks.so var/libhgks_nosplit.so var/libhgks_minb4.so var/libhgks_nosplit_minb4.so; do
  tag=$(basename $lib .so)
  timeout 300 env HGKS_LIB=$PWD/$lib python bench.py --steps 300 --warmup 5 --workload c2 --no-cpu-baseline > $O/bench_$tag.json 2>&1
  python -c "
import json
d=json.loads(open('$O/bench_$tag.json').read().strip().splitlines()[-1])
print('live $tag', '%.4g'%d['value'], round(d['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if v['launches'] and v['avg_ms']>0.03})"
  timeout 300 env HGKS_LIB=$PWD/$lib ncu --clock-control none --cache-control none --metrics gpu__time_duration.sum,launch__shared_mem_config_size,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers \
     -k regex:"k_flux|k_recon" --launch-skip 20 --launch-count 12 --csv python bench.py --workload c2 --steps 3 --warmup 8 --no-cpu-baseline > $O/ncu_$tag.csv 2> $O/ncu_$tag.err
  python - <<PY
import csv, collections
rows=[r for r in csv.reader(open('$O/ncu_$tag.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    agg[r[ki][:40]][r[mi]].append(r[vi])
for k,m in agg.items():
    t=[float(x.replace(',','')) for x in m['gpu__time_duration.sum']]
    print('  ncu $tag', k, 'us %.1f'%(sum(t)/len(t)/1e3 if max(t)>1e4 else sum(t)/len(t)), 'smem_cfg', set(m['launch__shared_mem_config_size']), 'warps%', m['sm__warps_active.avg.pct_of_peak_sustained_active'][:2])
PY
done
