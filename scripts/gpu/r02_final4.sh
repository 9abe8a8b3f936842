#!/bin/bash
# round-2 final verification on one B200 (after f4 and the late kernel changes): GPU suite,
# smoke, bench lines (default + reference arm + other workloads), ncu launch list and full
# captures (exported to CSV on the box: gpurun copies back at most 64 MiB), executed flop counts
O=gpurun_out/final4; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,clocks.max.mem,ecc.mode.current,power.limit --format=csv > $O/gpu.txt
nvidia-smi -q -d CLOCK,PERFORMANCE,ECC > $O/gpu_q.txt 2>&1
python -c "from paper_2407_00656_b200 import build as b; print('needs_build on the box:', b.needs_build())" > $O/lib.txt 2>&1
md5sum paper_2407_00656_b200/libhgks.so >> $O/lib.txt
timeout 1500 python -m pytest tests -q -m gpu --durations=30 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $O/bench_c5_200.json 2> $O/bench_c5_200.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python bench.py --workload c2 --steps 200 --warmup 5 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --workload c3 --steps 50 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --workload c3h --steps 50 --warmup 3 > $O/bench_c3h.json 2> $O/bench_c3h.err
timeout 900 python bench.py --workload c4 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --workload c2 --precision 32 --steps 200 --warmup 5 --no-cpu-baseline > $O/bench_c2_fp32.json 2> $O/bench_c2_fp32.err
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$B > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5.csv $B > /dev/null 2>&1
B2="python bench.py --workload c2 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$B2 > /dev/null 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_recon|k_flux|k_update" -c 5 -o /tmp/full_c2 -f $B2 > $O/ncu_full_c2.log 2>&1
ncu -i /tmp/full_c2.ncu-rep --page raw --csv > $O/ncu_full_c2.csv 2>/dev/null
ncu -i /tmp/full_c2.ncu-rep --page details --csv > $O/ncu_full_c2_details.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:"k_recon|k_flux" -c 3 -o /tmp/full_c5 -f $B > $O/ncu_full_c5.log 2>&1
ncu -i /tmp/full_c5.ncu-rep --page raw --csv > $O/ncu_full_c5.csv 2>/dev/null
B3="python bench.py --workload c3h --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none -k regex:"k_recon|k_flux" -c 4 -o /tmp/full_c3h -f $B3 > $O/ncu_full_c3h.log 2>&1
ncu -i /tmp/full_c3h.ncu-rep --page raw --csv > $O/ncu_full_c3h.csv 2>/dev/null
FL=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,gpu__time_duration.sum
for w in c2 c3; do for p in 64 32; do
  timeout 600 ncu --metrics $FL --clock-control none -k regex:"k_flux|k_recon" -c 8 --csv --log-file $O/flops_${w}_$p.csv $B2 --workload $w --precision $p > /dev/null 2>&1
done; done
gzip -f $O/*.csv
du -sh $O
ls -la $O
echo done
