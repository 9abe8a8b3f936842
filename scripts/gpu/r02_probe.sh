#!/bin/bash
# round-2 first GPU call: host facts, GPU suite, default bench line, oracle sizing probes
mkdir -p gpurun_out
{ nproc; free -g; lscpu | grep -i "model name"; nvidia-smi -L; } > gpurun_out/host.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench rc=$?" >> gpurun_out/bench_c5.err
timeout 1200 python scripts/oracle_probe.py c5 2 > gpurun_out/oracle_probe.log 2>&1
timeout 900 python scripts/oracle_probe.py c4 1 >> gpurun_out/oracle_probe.log 2>&1
timeout 600 python scripts/oracle_probe.py c3 1 >> gpurun_out/oracle_probe.log 2>&1
echo done
