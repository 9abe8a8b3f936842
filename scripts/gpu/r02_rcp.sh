# fast reciprocal / rsqrt (MUFU + Newton, no slow path) in the flux: parity subset + A/B
O=gpurun_out/rcp2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hybrid.py tests/test_gpu_multirank.py tests/test_gpu_fp32.py -x -q \
  -k "c1 or jittered or ragged or hex_box or stress or fallback or walled or kuhn_multirank or hybrid or prisms_only or t_stop or fp32_c1 or c2_size or bench_size or sphere_sub or sphere_sup or prandtl or dq0" > $O/tests.log 2>&1; tail -2 $O/tests.log
for round in 1 2; do
for w in c2 c5 c3; do
  steps=300; [ $w = c5 ] && steps=60; [ $w = c3 ] && steps=100
  for lib in paper_2407_00656_b200/libhgks.so var/libhgks_divrcp.so; do
    tag=$(basename $lib .so)
    timeout 300 env HGKS_LIB=$PWD/$lib python bench.py --steps $steps --warmup 5 --workload $w --no-cpu-baseline > $O/bench_${w}_${tag}_$round.json 2>&1
    python -c "
import json
d=json.loads(open('$O/bench_${w}_${tag}_$round.json').read().strip().splitlines()[-1])
print('$w $tag $round', '%.4g'%d['value'], round(d['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if v['launches'] and v['avg_ms']>0.03}, {k:round(v['frac'],3) for k,v in d['rooflines'].items()})"
  done
done
done
