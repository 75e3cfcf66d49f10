#!/usr/bin/env bash
# One gpurun call: GPU test suite (engine checkpoints kept for the CPU-side
# reference resume test), then the default bench line and the reference arm.
#   gpurun --timeout 3000 -- bash scripts/gpu_check.sh [tests|bench|all] [pytest -k expr]
set -u
what=${1:-all}
kexpr=${2:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
if [[ $what == tests || $what == all ]]; then
  args=(tests -m gpu -q -p no:cacheprovider --timeout 1800)
  [[ -n $kexpr ]] && args+=(-k "$kexpr")
  OGCP_ENGINE_CKPT_OUT=gpurun_out/engine_ckpt timeout 2400 python -m pytest "${args[@]}" -s \
    > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  tail -n 5 gpurun_out/pytest_gpu.log
fi
if [[ $what == bench || $what == all ]]; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json
  timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err
  echo "ref rc=$?"; tail -c 2000 gpurun_out/ref.json
fi
