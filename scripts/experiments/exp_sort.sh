# Zero-row sort experiment: parity tests touching the bucketed walk, A/B of the c4
# bench, and one ncu --set full capture of k_sgrad / k_wgrad with the sort on.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -s \
   -k "c4 or checkpoint_schema or bucket or shard or merged or stream" > gpurun_out/pytest_sort.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_sort.log; tail -n 3 gpurun_out/pytest_sort.log
bash scripts/ab_bench.sh "OGCP_SORT_ZEROS=0" "OGCP_SORT_ZEROS=1" "OGCP_SORT_ZEROS=0" "OGCP_SORT_ZEROS=1" | tee gpurun_out/ab_sort.txt
for k in k_sgrad k_wgrad; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 30 -c 1 -o gpurun_out/$k \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_$k.log 2>&1
  ncu -i gpurun_out/$k.ncu-rep --page raw --csv > gpurun_out/$k.raw.csv
  rm -f gpurun_out/$k.ncu-rep
done
python scripts/ncu_summary.py gpurun_out/k_sgrad.raw.csv; python scripts/ncu_summary.py gpurun_out/k_wgrad.raw.csv
