# Every SURVEY 8(d) config on one B200 (c4 is bench.py): one JSON line each -> gpurun_out/configs.jsonl
set -e
mkdir -p gpurun_out
{
  python scripts/stream_bench.py --config c1 --slices 6 2>/dev/null | tail -1
  python scripts/stream_bench.py --config c2 --slices 10 2>/dev/null | tail -1
  python scripts/config_bench.py c3 2>/dev/null | tail -1
  python scripts/config_bench.py c3 --semi 2>/dev/null | tail -1
  for r in 16 32 64 128; do python scripts/config_bench.py c5 --rank $r --slices 1 2>/dev/null | tail -1; done
} > gpurun_out/configs.jsonl
cat gpurun_out/configs.jsonl
