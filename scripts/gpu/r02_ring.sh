# per-thread cp.async ring for the P_0 operators: parity + A/B
O=gpurun_out/ring
mkdir -p $O
for D in 3; do
  HGKS_LIB=$PWD/var/libhgks_ring$D.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hybrid.py -x -q -k "c1_ten or jittered or hex_box_ten or hybrid_ten or sphere_sub" > $O/tests_ring$D.log 2>&1; tail -2 $O/tests_ring$D.log
done
for round in 1 2; do
for w in c2 c5 c3; do
  steps=300; [ $w = c5 ] && steps=60; [ $w = c3 ] && steps=100
  for lib in paper_2407_00656_b200/libhgks.so var/libhgks_ring2.so var/libhgks_ring3.so var/libhgks_ring4.so; do
    tag=$(basename $lib .so)
    timeout 300 env HGKS_LIB=$PWD/$lib python bench.py --steps $steps --warmup 5 --workload $w --no-cpu-baseline > $O/bench_${w}_${tag}_$round.json 2>&1
    python -c "
import json
d=json.loads(open('$O/bench_${w}_${tag}_$round.json').read().strip().splitlines()[-1])
print('$w $tag $round', '%.4g'%d['value'], round(d['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if v['launches'] and v['avg_ms']>0.03})"
  done
done
done
