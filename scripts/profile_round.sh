# Round measurement on one B200 (each ncu run only after the same command exited 0 without ncu):
#   1. the default bench line (e2e + cpu baseline)
#   2. an ncu launch list (gpu__time_duration per launch) over one step window
#   3. `ncu --set full` of one factor iteration's K3 walk (2 launches) and one weight walk
#      -> gpurun_out/roofline.raw.csv -> profiles/traffic.json (scripts/roofline.py)
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/pre.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 900 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/ncu_launches.log 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches.txt
# K3: the launches after 100 weight iterations of the first timed slice are factor-iteration walks
ncu --set full --clock-control none --import-source on -k regex:"k_walk_tma|k_sgrad" -s 610 -c 2 \
    -o gpurun_out/k3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_k3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_wgrad" -s 350 -c 1 \
    -o gpurun_out/k2w python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_k2w.log 2>&1
ncu -i gpurun_out/k3.ncu-rep --page raw --csv > gpurun_out/k3.raw.csv
ncu -i gpurun_out/k2w.ncu-rep --page raw --csv > gpurun_out/k2w.raw.csv
ncu -i gpurun_out/k3.ncu-rep --page source --csv --print-source sass > gpurun_out/k3.sass.csv 2>/dev/null || true
python - <<'PY'
import csv, io
a = open("gpurun_out/k3.raw.csv").read().splitlines()
b = open("gpurun_out/k2w.raw.csv").read().splitlines()
# same metric set (--set full): header + units from the first, data rows from both
ha, hb = next(csv.reader([a[0]])), next(csv.reader([b[0]]))
rows = [ha, next(csv.reader([a[1]]))] + [next(csv.reader([x])) for x in a[2:]]
for x in b[2:]:
    r = next(csv.reader([x]))
    d = dict(zip(hb, r))
    rows.append([d.get(k, "") for k in ha])
out = io.StringIO()
csv.writer(out).writerows(rows)
open("gpurun_out/roofline.raw.csv", "w").write(out.getvalue())
PY
python scripts/roofline.py gpurun_out/roofline.raw.csv > gpurun_out/traffic.json
python scripts/ncu_summary.py gpurun_out/roofline.raw.csv > gpurun_out/ncu_summary.txt
rm -f gpurun_out/k3.ncu-rep gpurun_out/k2w.ncu-rep
