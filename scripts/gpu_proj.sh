mkdir -p gpurun_out
timeout 1500 python scripts/shard_projection.py 1 2 4 8 > gpurun_out/shard_projection.txt 2> gpurun_out/shard_projection.err
echo "projection rc=$?"; cat gpurun_out/shard_projection.txt; tail -n 3 gpurun_out/shard_projection.err
bash scripts/prof_shard_step.sh
