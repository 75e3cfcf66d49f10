mkdir -p gpurun_out
for v in 0 1 0 1; do
  OGCP_DRAW_STAGE_ALWAYS=$v python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]);print('stage_always=$v', round(d['ms_per_step'],1), d['kernel_ms']['sgrad'], d['kernel_ms']['wgrad'])"
done
for v in 0 1; do
  OGCP_DRAW_STAGE_ALWAYS=$v timeout 900 python scripts/shard_projection.py 8 > gpurun_out/proj8_$v.txt 2>/dev/null
  echo "stage_always=$v"; cat gpurun_out/proj8_$v.txt | head -1
done
