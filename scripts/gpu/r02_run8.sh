#!/bin/bash
O=gpurun_out/r8; mkdir -p $O
timeout 600 env HGKS_RECON_PAIR=1 python -m pytest tests -q -m gpu -x -k "c1 or jittered or ragged or hex_box or stress or sphere or walled or fallback or dq0 or prandtl or lane_pair" > $O/pytest_pair.log 2>&1; echo "rc=$?" >> $O/pytest_pair.log
for i in 1 2; do
for rp in 0 1; do
HGKS_RECON_PAIR=$rp python bench.py --workload c2 --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $O/bench_c2_pair$rp\_$i.json 2>&1
done
HGKS_RECON_PAIR=1 HGKS_LIB=$PWD/paper_2407_00656_b200/libhgks_nodsplit.so python bench.py --workload c2 --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $O/bench_c2_pairold_$i.json 2>&1
done
HGKS_RECON_PAIR=1 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/bench_c5_pair1.json 2>&1
HGKS_RECON_PAIR=0 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/bench_c5_pair0.json 2>&1
for rp in 0 1; do HGKS_RECON_PAIR=$rp python bench.py --workload c3 --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/bench_c3_pair$rp.json 2>&1; done
python bench.py --workload c2 --precision 32 --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $O/bench_c2_fp32_dsplit.json 2>&1
HGKS_LIB=$PWD/paper_2407_00656_b200/libhgks_nodsplit.so python bench.py --workload c2 --precision 32 --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $O/bench_c2_fp32_old.json 2>&1
echo done
