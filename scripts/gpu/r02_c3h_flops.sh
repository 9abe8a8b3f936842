# executed FP64 op counts of the c3h (hybrid sphere) flux kernels, for bench.py's c3h flux rooflines
O=gpurun_out/c3hfl
mkdir -p $O
FL=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum
B="python bench.py --workload c3h --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$B > /dev/null 2>&1 && timeout 600 ncu --metrics $FL --clock-control none -k regex:"k_flux" -c 12 --csv --log-file $O/flops_c3h_64.csv $B > /dev/null 2>&1
ls -la $O
