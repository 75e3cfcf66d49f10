mkdir -p gpurun_out
for lib in paper_2110_14514_b200/libogcp_b200.so build/var/lib_minb3.so build/var/lib_minb4.so paper_2110_14514_b200/libogcp_b200.so build/var/lib_minb3.so; do
  OGCP_LIB=$lib python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$lib', round(d['ms_per_step'],1), d['kernel_ms']['sgrad'], d['kernel_ms']['wgrad'])"
done
