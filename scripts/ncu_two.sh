# ncu --set full of one k_sgrad and one k_wgrad launch inside the c4 bench (bucketed merged sets)
set -e
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/pre.json 2>/dev/null
for k in k_sgrad k_wgrad; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 30 -c 1 -o gpurun_out/$k \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_$k.log 2>&1 || true
done
OGCP_BUCKETS=0 ncu --set full --clock-control none -k regex:k_sgrad -s 30 -c 1 -o gpurun_out/k_sgrad_nob \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_nob.log 2>&1 || true

for r in gpurun_out/*.ncu-rep; do ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv; done
rm -f gpurun_out/k_sgrad_nob.ncu-rep gpurun_out/k_wgrad.ncu-rep
