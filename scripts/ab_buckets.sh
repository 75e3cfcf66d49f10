for lib in libogcp_b200 libogcp_b200_v1 libogcp_b200_v2 libogcp_b200_v3 libogcp_b200_v4; do
  OGCP_LIB=paper_2110_14514_b200/$lib.so OGCP_DEBUG_TIMING=1 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$lib', round(d['value']/1e9,3), d['ms_per_step'])"
  grep "timing\] solve" gpurun_out/ab.err | tail -2 | tr '\n' ' '; echo
done
