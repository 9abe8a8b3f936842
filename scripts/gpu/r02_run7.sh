#!/bin/bash
O=gpurun_out/r7; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x -k "not full_size and not c3_size and not bench_size and not table3" > $O/pytest_quick.log 2>&1; echo "rc=$?" >> $O/pytest_quick.log
for i in 1 2; do
for v in "" _notma _tmau2 _tmau7; do
HGKS_LIB=$PWD/paper_2407_00656_b200/libhgks$v.so python bench.py --workload c2 --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $O/bench_c2$v\_$i.json 2>&1
done; done
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 5 > $O/bench_c5.json 2>&1
HGKS_LIB=$PWD/paper_2407_00656_b200/libhgks_notma.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 5 > $O/bench_c5_notma.json 2>&1
B2="python bench.py --workload c2 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
ncu --set full --import-source on --clock-control none -k regex:"k_recon" -c 1 -o $O/full_recon -f $B2 > $O/ncu_recon.log 2>&1
echo done
