# Word-range sharded draws on one B200: the exact shard simulation (partition and
# gradient-sum tests, c4-scale bincount partition), the NCCL selftest, then the
# shard projection (rank-0 share measured, collectives modeled).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_shard.py tests/test_gpu_c4_draw.py -q -p no:cacheprovider -x \
   > gpurun_out/pytest_shard.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_shard.log; tail -n 15 gpurun_out/pytest_shard.log
timeout 1200 python scripts/shard_projection.py 1 2 4 8 > gpurun_out/shard_projection.txt 2> gpurun_out/shard_projection.err
echo "projection rc=$?"; cat gpurun_out/shard_projection.txt; tail -n 5 gpurun_out/shard_projection.err
