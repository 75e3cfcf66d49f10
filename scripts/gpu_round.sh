# Full round check on one B200: GPU test suite, profile_round (bench + launch list + roofline
# capture), reference arm, sanitizer.
mkdir -p gpurun_out
OGCP_ENGINE_CKPT_OUT=gpurun_out/engine_ckpt timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider \
   --timeout 1800 -s > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -n 3 gpurun_out/pytest_gpu.log
bash scripts/profile_round.sh; echo "profile rc=$?"
tail -c 2500 gpurun_out/bench.json; cat gpurun_out/launches.txt | head -25; cat gpurun_out/ncu_summary.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err
echo "ref rc=$?"
bash scripts/sanitize.sh
