# persistent k_recon (next-tile L2 prefetch) and persistent pipelined tau = 0 flux: parity + A/B
O=gpurun_out/p1
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp32.py tests/test_gpu_multirank.py tests/test_gpu_hybrid.py -x -q \
  -k "c1 or jittered or ragged or hex_box or stress or fallback or walled or fp32_c1 or kuhn_multirank or hybrid_ten or hybrid_density or prisms_only or t_stop or graph" > $O/tests.log 2>&1; tail -3 $O/tests.log
for w in c2 c5; do
  for v in new old_recon old_flux old_both; do
    case $v in
      new) E="";; old_recon) E="HGKS_RECON_GRID=tiles";; old_flux) E="HGKS_FLUX_PERSIST=0";; old_both) E="HGKS_RECON_GRID=tiles HGKS_FLUX_PERSIST=0";;
    esac
    steps=200; [ $w = c5 ] && steps=40
    env $E timeout 300 python bench.py --steps $steps --warmup 5 --workload $w --no-cpu-baseline > $O/bench_${w}_$v.json 2>&1
    python -c "
import json
d=json.loads(open('$O/bench_${w}_$v.json').read().strip().splitlines()[-1])
print('$w $v', '%.4g'%d['value'], round(d['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if v['launches'] and v['avg_ms']>0.03}, {k:round(v['frac'],3) for k,v in d['rooflines'].items()})"
  done
done
