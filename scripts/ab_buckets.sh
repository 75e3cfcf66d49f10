python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for r in 64 128; do python scripts/config_bench.py c5 --rank $r --slices 1 2>&1 | tail -1; done
