# ldr 32 Grams: tcgen05 with the decoupled raw ring (k_gram_umma32) vs mma.sync (k_gram_tc<32>):
# parity tests, then the c4 bench step (bench.py OGCP_UMMA_GRAM=0: mma.sync).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_coverage.py -q -p no:cacheprovider -k "grams" > gpurun_out/pytest_gram.log 2>&1
echo "pytest rc=$?"; tail -n 3 gpurun_out/pytest_gram.log
for v in 1 0 1 0; do
  OGCP_UMMA_GRAM=$v python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('umma=$v', round(d['ms_per_step'],1), d['kernel_ms']['gram'], d['kernel_ms']['sgrad'])"
done
bash scripts/experiments/ncu_gram32.sh
