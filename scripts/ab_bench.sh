# A/B the c4 bench across environment settings (engine knobs such as OGCP_BUCKETS,
# OGCP_MERGE, OGCP_SPLIT, or OGCP_LIB=<variant .so>): one line per setting with
# entries/s, ms per step and the per-launch k_sgrad / k_wgrad times.
#   bash scripts/ab_bench.sh "OGCP_BUCKETS=1" "OGCP_BUCKETS=4"
for cfg in "$@"; do
  env $cfg python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab.json 2> gpurun_out/ab.err
  python - "$cfg" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
k, n = d["kernel_ms"], d["kernel_launch_brackets"]
print(sys.argv[1], round(d["value"] / 1e9, 3), d["ms_per_step"], round(k["sgrad"] / n["sgrad"], 3),
      round(k["wgrad"] / n["wgrad"], 3))
PY
done
