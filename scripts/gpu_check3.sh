mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_shard.py tests/test_gpu_c4_draw.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/pytest_sub.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_sub.log; tail -n 4 gpurun_out/pytest_sub.log
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
python -c "import json;d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['kernel_ms'],d['roofline']['avg_launch_ms'],d['roofline']['frac'],d['roofline']['l2_frac'])"
timeout 1500 python scripts/shard_projection.py 1 2 4 8 > gpurun_out/shard_projection.txt 2> gpurun_out/shard_projection.err
echo "projection rc=$?"; cat gpurun_out/shard_projection.txt; tail -n 3 gpurun_out/shard_projection.err
