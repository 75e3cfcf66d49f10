python -m pytest tests -m gpu -q -x 2>&1 | tail -1
python scripts/stream_bench.py --config c1 --slices 6 2>&1 | tail -1
python scripts/stream_bench.py --config c2 --slices 10 2>&1 | tail -1
