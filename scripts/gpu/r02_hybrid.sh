# f4 hybrid meshes: GPU parity + regression subset + C2 bench (round 2)
O=gpurun_out/h1
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hybrid.py -q > $O/hybrid.log 2>&1; tail -15 $O/hybrid.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp32.py tests/test_gpu_multirank.py -x -q -k "c1 or hex or walled or sphere_residual or kuhn_multirank or fp32_c1 or ragged" > $O/regress.log 2>&1; tail -3 $O/regress.log
timeout 300 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline > $O/bench_c2.json 2>&1; tail -c 600 $O/bench_c2.json
