# source-level (SASS) stall profile of the tau = 0 flux and the reconstruction on C2
O=gpurun_out/src
mkdir -p $O
python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > $O/plain.log 2>&1 || { tail -5 $O/plain.log; exit 1; }
for k in k_flux k_recon; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^${k}" --launch-skip 4 --launch-count 1 \
     -o /tmp/$k python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_$k.log 2>&1
  ncu -i /tmp/$k.ncu-rep --page source --csv --print-source sass > /tmp/${k}_sass.csv 2>> $O/ncu_$k.log
  ncu -i /tmp/$k.ncu-rep --page details --csv > /tmp/${k}_details.csv 2>> $O/ncu_$k.log
  gzip -c /tmp/${k}_sass.csv > $O/${k}_sass.csv.gz
  gzip -c /tmp/${k}_details.csv > $O/${k}_details.csv.gz
  ls -la /tmp/${k}*
done
