# pipelined tau = 0 flux (two-stage TMA pipeline per warp): parity subset + A/B vs k_flux (env switch)
O=gpurun_out/pipe
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hybrid.py tests/test_gpu_multirank.py tests/test_gpu_fp32.py -x -q \
  -k "c1 or jittered or ragged or hex_box or stress or fallback or walled or kuhn_multirank or hybrid_ten or prisms_only or t_stop or fp32_c1 or c2_size or bench_size or graph" > $O/tests.log 2>&1; tail -2 $O/tests.log
for round in 1 2; do
for w in c2 c5; do
  steps=300; [ $w = c5 ] && steps=60
  for v in 1 0; do
    timeout 300 env HGKS_FLUX_PIPE=$v python bench.py --steps $steps --warmup 5 --workload $w --no-cpu-baseline > $O/bench_${w}_pipe${v}_$round.json 2>&1
    python -c "
import json
d=json.loads(open('$O/bench_${w}_pipe${v}_$round.json').read().strip().splitlines()[-1])
print('$w pipe$v $round', '%.4g'%d['value'], round(d['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if v['launches'] and v['avg_ms']>0.03}, {k:round(v['frac'],3) for k,v in d['rooflines'].items()})"
  done
done
done
