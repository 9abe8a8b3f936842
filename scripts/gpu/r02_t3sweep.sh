#!/bin/bash
# T3 reading study: dQ0 readings x CFL, N = 10..80, on the GPU path
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "dq0 or fallback or t_stop or loopback" > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
for mode in 0 1 2; do for cfl in 0.3 0.5 0.7; do
  timeout 600 python scripts/convergence_gpu.py --N 10 20 40 80 --cfl $cfl --dq0-mode $mode >> gpurun_out/t3sweep.jsonl 2>> gpurun_out/t3sweep.err
done; done
echo done
