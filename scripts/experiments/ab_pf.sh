mkdir -p gpurun_out
for lib in paper_2110_14514_b200/libogcp_b200.so build/var/lib_nopf.so paper_2110_14514_b200/libogcp_b200.so build/var/lib_nopf.so; do
  OGCP_LIB=$lib python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$lib', round(d['ms_per_step'],1), d['kernel_ms']['sgrad'], d['kernel_ms']['wgrad'], d['kernel_ms']['objective'])"
done
for lib in paper_2110_14514_b200/libogcp_b200.so build/var/lib_nopf.so; do
  for c in c1 c2; do OGCP_LIB=$lib python scripts/stream_bench.py --config $c --slices 60 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['config'], round(d['ms_per_slice'],2), d['max_rel_sampled_fit_vs_reference'])"; done
done
