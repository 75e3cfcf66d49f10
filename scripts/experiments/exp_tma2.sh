mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -s -x \
   -k "dense_draw or shard or c4 or stream" > gpurun_out/pytest_tma2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_tma2.log; tail -n 3 gpurun_out/pytest_tma2.log
bash scripts/ab_bench.sh "OGCP_TMA=2" "OGCP_TMA=1" "OGCP_TMA=0" "OGCP_TMA=1" | tee gpurun_out/ab_tma2.txt
ncu --set full --clock-control none -k regex:"k_walk_tma" -s 610 -c 2 -o gpurun_out/k3b \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_k3b.log 2>&1
ncu -i gpurun_out/k3b.ncu-rep --page raw --csv > gpurun_out/k3b.raw.csv; rm -f gpurun_out/k3b.ncu-rep
python scripts/roofline.py gpurun_out/k3b.raw.csv > gpurun_out/traffic_k3b.json
python scripts/ncu_summary.py gpurun_out/k3b.raw.csv
python -c "
import json; d=json.load(open('gpurun_out/traffic_k3b.json'))
for k,w in d['walks'].items(): print(k, w['time_ms'], w['dram_bytes']/1e9, w['l2_bytes']/1e9, w['l2_bytes']/w['time_ms']/1e6, 'GB/s L2')"
