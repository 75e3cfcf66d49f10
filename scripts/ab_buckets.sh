for cfg in "OGCP_X=1" "OGCP_SIDE_PRIO_HIGH=1"; do
  env $cfg python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$cfg', round(d['value']/1e9,3), d['ms_per_step'])"
  env $cfg python scripts/config_bench.py c5 --rank 128 --slices 1 2>&1 | tail -1 | cut -c1-120
done
