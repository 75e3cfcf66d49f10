python -m pytest tests -m gpu -q -x 2>&1 | tail -1
python scripts/stream_bench.py --config c1 --slices 6 2>&1 | tail -1
python scripts/stream_bench.py --config c2 --slices 10 2>&1 | tail -1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print(round(d['value']/1e9,3), d['ms_per_step'])"
