for cfg in "OGCP_NO_FILTER=1 OGCP_GPAD_KB=0" "OGCP_NO_FILTER=1 OGCP_GPAD_KB=2048" "OGCP_NO_FILTER=1 OGCP_GPAD_KB=65536" "OGCP_NO_FILTER=1 OGCP_GPAD_KB=1024" "OGCP_NO_FILTER=1 OGCP_GPAD_KB=4096" "OGCP_NO_FILTER=1 OGCP_GPAD_KB=16384"; do
  env $cfg python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernel_ms']; n=d['kernel_launch_brackets']
print('$cfg', round(d['value']/1e9,3), {c: round(k[c]/max(n[c],1),3) for c in k})"
done
