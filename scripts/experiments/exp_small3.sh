mkdir -p gpurun_out
for c in c1 c2; do timeout 600 python scripts/stream_bench.py --config $c; done | tee gpurun_out/small3.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 2000 --csv --log-file gpurun_out/launches_c1.csv \
   python scripts/stream_bench.py --config c1 --slices 2 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_c1.csv | head -12
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 2000 --csv --log-file gpurun_out/launches_c2.csv \
   python scripts/stream_bench.py --config c2 --slices 3 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_c2.csv | head -16
