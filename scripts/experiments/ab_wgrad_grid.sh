# c4: k_wgrad with its full grid (2 CTAs per SM) vs half (one per SM, leaving room for the side-stream draw).
# (needs the OGCP_WGRAD_GRID_DIV switch, removed after this experiment: k_wgrad grid / div)
mkdir -p gpurun_out
for v in 1 2 1 2; do
  OGCP_WGRAD_GRID_DIV=$v python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('div=$v', round(d['ms_per_step'],1), d['kernel_ms']['wgrad'], d['kernel_ms']['sgrad'], round(d['draw_side_stream_wall_ms'],1))"
done
