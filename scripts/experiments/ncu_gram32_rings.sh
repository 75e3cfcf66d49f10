# k_gram_umma32 ring depths (transposed stages, raw stages): device time per launch.
mkdir -p gpurun_out
for lib in paper_2110_14514_b200/libogcp_b200.so build/var/lib_g32_5_4.so build/var/lib_g32_3_6.so build/var/lib_g32_5_3.so; do
  OGCP_LIB=$lib ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_gram_umma32" -s 30 -c 12 --csv \
      --log-file gpurun_out/g.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
  echo "$lib"; python scripts/launch_summary.py gpurun_out/g.csv | sed -n 2p
done
