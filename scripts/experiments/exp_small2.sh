mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -s -x -k "stream or static or gaussian or coverage or parity" > gpurun_out/pytest_small.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_small.log; tail -n 3 gpurun_out/pytest_small.log
for c in c1 c2; do timeout 600 python scripts/stream_bench.py --config $c --profile; done | tee gpurun_out/small2.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none -s 20000 -c 3000 --csv --log-file gpurun_out/launches_c2b.csv \
   python scripts/stream_bench.py --config c2 --slices 3 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_c2b.csv | head -20
