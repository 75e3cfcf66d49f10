mkdir -p gpurun_out
python scripts/shard_step.py 8 > gpurun_out/shard_step8.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_n8.csv python scripts/shard_step.py 8 > gpurun_out/ncu_n8.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_n8.csv > gpurun_out/launches_n8.txt
cat gpurun_out/shard_step8.log; head -45 gpurun_out/launches_n8.txt; tail -3 gpurun_out/ncu_n8.log
