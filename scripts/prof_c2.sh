mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -s 20000 -c 2000 --csv \
    --log-file gpurun_out/launches_c2.csv python scripts/stream_bench.py --config c2 --slices 20 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_c2.csv > gpurun_out/launches_c2.txt; head -16 gpurun_out/launches_c2.txt
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches_c2.csv')))
hi=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[hi]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
seq=[(r[ki].split('(')[0].replace('void ',''), r[vi]) for r in rows[hi+1:hi+41] if len(r)>vi]
for s in seq: print(s)
PY
