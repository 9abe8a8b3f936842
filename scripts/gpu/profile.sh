# Round profile capture on one B200 (run under gpurun).  Outputs -> gpurun_out/prof/
set -x
O=gpurun_out/prof; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
tools/microbench/fp64_peak > $O/peaks.json 2>&1
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
# each command first runs clean (exit 0), then under ncu
$B > $O/bench_c2.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv $B > /dev/null 2>&1
$B > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_recon|k_flux|k_update" -c 6 -o $O/full_c2 -f $B > $O/ncu_full_c2.log 2>&1
FL=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,gpu__time_duration.sum
for w in c2 c3; do for p in 64 32; do
  $B --workload $w --precision $p > /dev/null 2>&1 && \
  ncu --metrics $FL --clock-control none -k regex:"k_flux|k_recon" -c 8 --csv --log-file $O/flops_${w}_$p.csv $B --workload $w --precision $p > /dev/null 2>&1
done; done
$B --workload c3 > $O/bench_c3.json 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_flux|k_recon" -c 2 -o $O/full_c3 -f $B --workload c3 > $O/ncu_full_c3.log 2>&1
ls -la $O
