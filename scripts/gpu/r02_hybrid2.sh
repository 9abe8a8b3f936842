# f4: hybrid sphere parity (small + bench size) and the c3h bench line
O=gpurun_out/h2
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_hybrid.py -q -k "sphere or c3h" > $O/hybrid_sphere.log 2>&1; tail -5 $O/hybrid_sphere.log
timeout 600 python bench.py --steps 100 --warmup 5 --workload c3h > $O/bench_c3h.json 2>&1; tail -c 400 $O/bench_c3h.json
timeout 600 python bench.py --steps 100 --warmup 5 --workload c3 --no-cpu-baseline > $O/bench_c3.json 2>&1; tail -c 200 $O/bench_c3.json
