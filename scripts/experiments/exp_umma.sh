mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_coverage.py -m gpu -q -p no:cacheprovider -x -k "tensor_core_grams or 130 or weights" > gpurun_out/pytest_umma.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_umma.log; tail -n 15 gpurun_out/pytest_umma.log
for r in 64 128; do
  OGCP_UMMA=0 timeout 600 python scripts/config_bench.py c5 --rank $r --slices 1 2>&1 | tail -1
  timeout 600 python scripts/config_bench.py c5 --rank $r --slices 1 2>&1 | tail -1
done | tee gpurun_out/umma_c5.jsonl
