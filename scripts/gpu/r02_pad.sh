# address-mapping study: record / operator array offsets vs the recon / flux times (C2, C5)
O=gpurun_out/pad
mkdir -p $O
for w in c2 c5; do
  steps=200; [ $w = c5 ] && steps=40
  for pads in "0 0" "0 4" "0 64" "0 1028" "0 2048" "0 8196" "4 0" "64 0" "1028 0" "2048 0" "8196 0" "1028 1028"; do
    set -- $pads
    timeout 300 env HGKS_PAD_REC=$1 HGKS_PAD_OP=$2 python bench.py --steps $steps --warmup 5 --workload $w --no-cpu-baseline --e2e-steps 2 > $O/bench_${w}_$1_$2.json 2>&1
    python -c "
import json
d=json.loads(open('$O/bench_${w}_$1_$2.json').read().strip().splitlines()[-1])
print('$w rec+$1K op+$2K', '%.4g'%d['value'], round(d['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if v['launches'] and v['avg_ms']>0.03})"
  done
done
