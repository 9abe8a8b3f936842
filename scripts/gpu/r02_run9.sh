#!/bin/bash
O=gpurun_out/r9; mkdir -p $O
for i in 1 2; do
for v in "" _carve25 _carve50 _carve75 _carve100; do
HGKS_LIB=$PWD/paper_2407_00656_b200/libhgks$v.so python bench.py --workload c2 --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $O/bench_c2$v\_$i.json 2>&1
done; done
for v in "" _carve75 _carve100; do
HGKS_LIB=$PWD/paper_2407_00656_b200/libhgks$v.so python bench.py --workload c2 --precision 32 --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $O/bench_c2_fp32$v.json 2>&1
HGKS_LIB=$PWD/paper_2407_00656_b200/libhgks$v.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/bench_c5$v.json 2>&1
done
echo done
