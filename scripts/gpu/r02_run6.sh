#!/bin/bash
O=gpurun_out/r6; mkdir -p $O
for i in 1 2; do
for v in _oldrecon _neu4 _neu7 _neu14; do
HGKS_LIB=$PWD/paper_2407_00656_b200/libhgks$v.so python bench.py --workload c2 --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $O/bench_c2$v\_$i.json 2>&1
done; done
echo done
