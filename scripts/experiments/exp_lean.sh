# Lean 3-way walk kernels: parity tests on the merged paths, c4 A/B against the
# generic kernels, ncu --set full of k_sgrad3 / k_wgrad3 (nonzero walks).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -s \
   -k "dense_draw or shard or c4 or stream or semi or static or coverage" > gpurun_out/pytest_lean.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_lean.log; tail -n 4 gpurun_out/pytest_lean.log
bash scripts/ab_bench.sh "OGCP_LEAN=0" "OGCP_LEAN=1" "OGCP_LEAN=1 OGCP_SORT_ZEROS=1" | tee gpurun_out/ab_lean.txt
for k in k_sgrad3 k_wgrad3; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 30 -c 1 -o gpurun_out/$k \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_$k.log 2>&1
  ncu -i gpurun_out/$k.ncu-rep --page raw --csv > gpurun_out/$k.raw.csv
  ncu -i gpurun_out/$k.ncu-rep --page source --csv --print-source sass > gpurun_out/$k.sass.csv 2>/dev/null
  rm -f gpurun_out/$k.ncu-rep
done
python scripts/ncu_summary.py gpurun_out/k_sgrad3.raw.csv; python scripts/ncu_summary.py gpurun_out/k_wgrad3.raw.csv
ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 900 --csv \
    --log-file gpurun_out/launches_lean.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/ncu_launches_lean.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_lean.csv | head -30
