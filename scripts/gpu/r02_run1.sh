#!/bin/bash
# full GPU suite (with the full-size parity tests), default bench line, launch list, ncu capture
O=gpurun_out/r1; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu --durations=20 > $O/pytest_full.log 2>&1; echo "rc=$?" >> $O/pytest_full.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --workload c2 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$B > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5.csv $B > /dev/null 2>&1
B2="python bench.py --workload c2 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$B2 > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:"k_flux|k_recon" -c 3 -o $O/full_c2 -f $B2 > $O/ncu_full_c2.log 2>&1
FL=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum
ncu --metrics $FL --clock-control none -k regex:"k_flux|k_recon" -c 8 --csv --log-file $O/flops_c2_64.csv $B2 > /dev/null 2>&1
echo done
