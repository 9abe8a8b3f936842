# split-Horner erfc / exp_neg: parity subset + A/B against the single-chain build
O=gpurun_out/s1
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hybrid.py -x -q \
  -k "c1 or jittered or hex_box or stress or fallback or sphere_sub or sphere_residual or hybrid_ten or prandtl" > $O/tests.log 2>&1; tail -3 $O/tests.log
for round in 1 2; do
for w in c2 c5; do
  steps=300; [ $w = c5 ] && steps=60
  for lib in paper_2407_00656_b200/libhgks.so var/libhgks_nosplit.so; do
    tag=$(basename $lib .so)_$w_$round
    timeout 300 env HGKS_LIB=$PWD/$lib python bench.py --steps $steps --warmup 5 --workload $w --no-cpu-baseline > $O/bench_${w}_$(basename $lib .so)_$round.json 2>&1
    python -c "
import json
d=json.loads(open('$O/bench_${w}_$(basename $lib .so)_$round.json').read().strip().splitlines()[-1])
print('$w $(basename $lib .so) $round', '%.4g'%d['value'], round(d['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if v['launches'] and v['avg_ms']>0.03}, {k:round(v['frac'],3) for k,v in d['rooflines'].items()})"
  done
done
done
