# A/B matrix: lines of "LIB|ENV|bench args"; prints one summary line each
run() {
  lib=$1; envs=$2; shift 2
  tag=$(echo "$lib $envs $*" | tr ' =/|' '____')
  timeout 180 env HGKS_LIB=$PWD/$lib $envs python bench.py --steps 150 --warmup 10 --no-cpu-baseline "$@" > gpurun_out/ab_$tag.json 2>&1
  python -c "
import json
try:
  d=json.loads(open('gpurun_out/ab_$tag.json').read().strip().splitlines()[-1])
  print('$lib | $envs | $*', round(d['value']/1e6,1), round(d['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if v['launches'] and v['avg_ms']>0.03})
except Exception as e: print('$lib | $envs | $* FAILED', open('gpurun_out/ab_$tag.json').read()[-300:])"
}
B=paper_2407_00656_b200/libhgks.so
run $B "HGKS_FLUX_PERSISTENT=0" --workload c2
run $B "HGKS_FLUX_PERSISTENT=1" --workload c2
run $B "HGKS_FLUX_PAIR=1" --workload c2
run build_var_p5.so "HGKS_FLUX_PAIR=1" --workload c2
run build_var_p8.so "HGKS_FLUX_PAIR=1" --workload c2
run $B "HGKS_FLUX_PERSISTENT=0" --workload c3
run $B "HGKS_FLUX_PERSISTENT=1" --workload c3
run $B "HGKS_FLUX_MPAIR=1" --workload c3
run build_var_mp2.so "HGKS_FLUX_MPAIR=1" --workload c3
run build_var_mp4.so "HGKS_FLUX_MPAIR=1" --workload c3
run $B "HGKS_FLUX_PERSISTENT=1" --workload c2 --precision 32
run $B "HGKS_FLUX_PAIR=1" --workload c2 --precision 32
run $B "HGKS_FLUX_PERSISTENT=1" --workload c3 --precision 32
run $B "HGKS_FLUX_MPAIR=1" --workload c3 --precision 32
