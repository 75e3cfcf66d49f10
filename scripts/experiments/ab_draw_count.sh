# Draw passes of the zero stream: working tree vs the previous commit (build/var/lib_old.so):
# bit-exact draw tests, ncu device time of k_draw_count<3> / k_draw_write<3>, c4 bench steps.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c4_draw.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "draw" > gpurun_out/pytest_draw.log 2>&1
echo "pytest rc=$?"; tail -n 2 gpurun_out/pytest_draw.log
for lib in paper_2110_14514_b200/libogcp_b200.so build/var/lib_old.so; do
  OGCP_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_draw_(count|write)" -s 40 -c 20 --csv \
      --log-file gpurun_out/dc.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
  echo "$lib"; python scripts/launch_summary.py gpurun_out/dc.csv | sed -n 2,4p
done
bash scripts/experiments/ab_lib.sh
