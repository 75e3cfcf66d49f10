for cfg in "OGCP_GRID_PCT=100" "OGCP_GRID_PCT=90" "OGCP_GRID_PCT=80" "OGCP_GRID_PCT=65"; do
  env $cfg python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernel_ms']; n=d['kernel_launch_brackets']
print('$cfg', round(d['value']/1e9,3), d['ms_per_step'], {c: round(k[c]/max(n[c],1),3) for c in k})"
done
