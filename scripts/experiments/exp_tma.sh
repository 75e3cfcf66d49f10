# TMA-fed walks: parity on the merged paths, c4 A/B, ncu of the walk kernels.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -s -x \
   -k "dense_draw or shard or c4 or stream" > gpurun_out/pytest_tma.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_tma.log; tail -n 4 gpurun_out/pytest_tma.log
bash scripts/ab_bench.sh "OGCP_TMA=0" "OGCP_TMA=1" "OGCP_TMA=1 OGCP_SORT_ZEROS=1" | tee gpurun_out/ab_tma.txt
ncu --set full --clock-control none --import-source on -k regex:k_walk_tma -s 206 -c 2 -o gpurun_out/k_walk_tma \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_k_walk_tma.log 2>&1
ncu -i gpurun_out/k_walk_tma.ncu-rep --page raw --csv > gpurun_out/k_walk_tma.raw.csv
rm -f gpurun_out/k_walk_tma.ncu-rep
python scripts/ncu_summary.py gpurun_out/k_walk_tma.raw.csv
