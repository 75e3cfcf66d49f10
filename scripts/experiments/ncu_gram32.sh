# Device time of the c4 Grams (ldr 32) per launch: tcgen05 k_gram_umma32 vs mma.sync k_gram_tc<32>.
mkdir -p gpurun_out
for v in 1 0; do
  OGCP_UMMA_GRAM=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_gram" -s 30 -c 12 --csv \
      --log-file gpurun_out/gram_$v.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
  echo "umma=$v"; python scripts/launch_summary.py gpurun_out/gram_$v.csv | head -6
done
