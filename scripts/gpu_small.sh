# Small configs on one B200: stream parity tests, then c1 / c2 slices per second.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_streams.py tests/test_gpu_coverage.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/pytest_small.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_small.log; tail -n 3 gpurun_out/pytest_small.log
for c in c1 c2; do python scripts/stream_bench.py --config $c 2>/dev/null; done
