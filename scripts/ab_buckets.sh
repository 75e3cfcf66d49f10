for lib in libogcp_b200 libogcp_b200_s241 libogcp_b200; do
  OGCP_LIB=paper_2110_14514_b200/$lib.so python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernel_ms']; n=d['kernel_launch_brackets']
print('$lib', round(d['value']/1e9,3), d['ms_per_step'], round(k['sgrad']/n['sgrad'],3), round(k['wgrad']/n['wgrad'],3))"
done
