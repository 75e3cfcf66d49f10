mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_c4_draw.py tests/test_gpu_shard.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/pytest_sub.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_sub.log; tail -n 4 gpurun_out/pytest_sub.log
bash scripts/ab_lib.sh
