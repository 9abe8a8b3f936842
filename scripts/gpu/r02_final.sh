#!/bin/bash
# round-2 verification on one B200: GPU suite, smoke, bench lines (default + reference arm +
# other workloads), ncu launch list and full captures, the Prandtl-corrected sphere runs
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -q -m gpu --durations=25 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python bench.py --workload c2 --steps 200 --warmup 5 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --workload c3 --steps 50 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --workload c4 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --workload c2 --precision 32 --steps 200 --warmup 5 --no-cpu-baseline > $O/bench_c2_fp32.json 2> $O/bench_c2_fp32.err
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$B > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5.csv $B > /dev/null 2>&1
B2="python bench.py --workload c2 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
# ncu reports are exported to CSV on the box and deleted (gpurun copies back at most 64 MiB)
$B2 > /dev/null 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_recon|k_flux|k_update" -c 5 -o /tmp/full_c2 -f $B2 > $O/ncu_full_c2.log 2>&1
ncu -i /tmp/full_c2.ncu-rep --page raw --csv > $O/ncu_full_c2.csv 2>/dev/null
ncu -i /tmp/full_c2.ncu-rep --page details --csv > $O/ncu_full_c2_details.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:"k_recon|k_flux" -c 3 -o /tmp/full_c5 -f $B > $O/ncu_full_c5.log 2>&1
ncu -i /tmp/full_c5.ncu-rep --page raw --csv > $O/ncu_full_c5.csv 2>/dev/null
gzip -f $O/*.csv
FL=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,gpu__time_duration.sum
for w in c2 c3; do for p in 64 32; do
  timeout 600 ncu --metrics $FL --clock-control none -k regex:"k_flux|k_recon" -c 8 --csv --log-file $O/flops_${w}_$p.csv $B2 --workload $w --precision $p > /dev/null 2>&1
done; done
timeout 900 python scripts/sphere_wake.py --N 35 --ma 0.2535 --re 118 --prandtl 0.72 --t-end 70 > $O/wake_sub35_pr072.log 2>&1
timeout 900 python scripts/sphere_wake.py --N 35 --ma 1.5 --re 300 --prandtl 0.72 --t-end 36 > $O/wake_sup35_pr072.log 2>&1
timeout 1500 python scripts/sphere_wake.py --N 64 --ma 0.2535 --re 118 --prandtl 0.72 --t-end 70 > $O/wake_sub64_pr072.log 2>&1
du -sh $O
ls -la $O
echo done
