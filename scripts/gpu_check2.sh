# Full GPU suite, then the shard projection and the N=8 per-rank launch list.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -n 6 gpurun_out/pytest_gpu.log
timeout 1200 python scripts/shard_projection.py 1 2 4 8 > gpurun_out/shard_projection.txt 2> gpurun_out/shard_projection.err
echo "projection rc=$?"; cat gpurun_out/shard_projection.txt; tail -n 3 gpurun_out/shard_projection.err
bash scripts/prof_shard_step.sh
