for cfg in "OGCP_SORT_ZEROS=1 OGCP_ZSORT_BITS=8" "OGCP_SORT_ZEROS=1 OGCP_ZSORT_BITS=12" "OGCP_SORT_ZEROS=1 OGCP_ZSORT_BITS=16"; do
  env $cfg OGCP_DEBUG_TIMING=1 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernel_ms']; n=d['kernel_launch_brackets']
print('$cfg', round(d['value']/1e9,3), d['ms_per_step'], round(k['sgrad']/n['sgrad'],3), round(k['wgrad']/n['wgrad'],3))"
  grep "timing\] solve" gpurun_out/ab.err | tail -2 | tr '\n' ' '; echo
done
