# Round-end evidence on one B200: GPU suite (with engine checkpoints for the interop
# test), bench line + launch list + ncu K3/K2w roofline capture (profile_round.sh),
# the reference arm, every config, and the multi-GPU projection.
mkdir -p gpurun_out
bash scripts/gpu_round.sh
bash scripts/all_configs.sh > /dev/null 2>&1; echo "configs rc=$?"; cat gpurun_out/configs.jsonl
timeout 1500 python scripts/shard_projection.py 1 2 4 8 > gpurun_out/shard_projection.txt 2> gpurun_out/shard_projection.err
echo "projection rc=$?"; cat gpurun_out/shard_projection.txt
