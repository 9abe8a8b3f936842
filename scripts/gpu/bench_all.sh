# Bench lines for profiles/: default (C2 fp64 with CPU baseline), reference arm, C3, C4, FP32.
O=gpurun_out/lines; mkdir -p $O
python bench.py > $O/c2.json 2> $O/c2.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/reference.json 2> $O/reference.err
python bench.py --precision 32 --no-cpu-baseline > $O/c2_fp32.json 2> $O/c2_fp32.err
python bench.py --workload c3 --steps 200 > $O/c3.json 2> $O/c3.err
python bench.py --workload c3 --steps 200 --precision 32 > $O/c3_fp32.json 2> $O/c3_fp32.err
python bench.py --workload c4 --steps 50 > $O/c4.json 2> $O/c4.err
for f in $O/*.json; do echo $f; tail -c 400 $f; echo; done
python bench.py --workload c5 --steps 50 --no-cpu-baseline > $O/c5.json 2> $O/c5.err
