# TMA bulk record staging + constant-bank exp coefficients: parity subset + A/B vs cp.async staging
O=gpurun_out/tma2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hybrid.py tests/test_gpu_multirank.py tests/test_gpu_fp32.py -x -q \
  -k "c1 or jittered or ragged or hex_box or stress or fallback or walled or kuhn_multirank or hybrid_ten or prisms_only or sphere_sub or t_stop or fp32_c1 or c2_size or bench_size" > $O/tests.log 2>&1; tail -2 $O/tests.log
for round in 1 2; do
for w in c2 c5; do
  steps=300; [ $w = c5 ] && steps=60
  for lib in paper_2407_00656_b200/libhgks.so var/libhgks_nodedup.so var/libhgks_notma.so; do
    tag=$(basename $lib .so)
    timeout 300 env HGKS_LIB=$PWD/$lib python bench.py --steps $steps --warmup 5 --workload $w --no-cpu-baseline > $O/bench_${w}_${tag}_$round.json 2>&1
    python -c "
import json
d=json.loads(open('$O/bench_${w}_${tag}_$round.json').read().strip().splitlines()[-1])
print('$w $tag $round', '%.4g'%d['value'], round(d['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if v['launches'] and v['avg_ms']>0.03}, {k:round(v['frac'],3) for k,v in d['rooflines'].items()})"
  done
done
done
python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^k_flux" --launch-skip 4 --launch-count 1 -o /tmp/kf python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu.log 2>&1
ncu -i /tmp/kf.ncu-rep --page source --csv --print-source sass > /tmp/kf_sass.csv 2>> $O/ncu.log
ncu -i /tmp/kf.ncu-rep --page raw --csv > /tmp/kf_raw.csv 2>> $O/ncu.log
gzip -c /tmp/kf_sass.csv > $O/k_flux_tau0_s1_tma2_sass.csv.gz; gzip -c /tmp/kf_raw.csv > $O/k_flux_tau0_s1_tma2_raw.csv.gz
