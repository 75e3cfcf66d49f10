# c1 / c2 per-kernel launch lists (a window of one stream's steady state).
mkdir -p gpurun_out
for c in c1 c2; do
  python scripts/stream_bench.py --config $c --slices 20 --profile > gpurun_out/sb_$c.json 2>&1; cat gpurun_out/sb_$c.json
  ncu --metrics gpu__time_duration.sum --clock-control none -s 20000 -c 3000 --csv \
      --log-file gpurun_out/launches_$c.csv python scripts/stream_bench.py --config $c --slices 20 > /dev/null 2>&1
  python scripts/launch_summary.py gpurun_out/launches_$c.csv > gpurun_out/launches_$c.txt; head -25 gpurun_out/launches_$c.txt
done
