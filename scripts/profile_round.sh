# Round measurement on one B200: the default bench line (e2e + cpu baseline), an ncu launch
# list (per-kernel durations, a window of one step) and one `ncu --set full` capture of each
# sample kernel (k_sgrad, k_wgrad) exported as raw CSV.  Each ncu run only after the same
# command exited 0 without ncu.
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/pre.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 800 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/ncu_launches.log 2>&1
for k in k_sgrad k_wgrad; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 30 -c 1 -o gpurun_out/$k \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_$k.log 2>&1
  ncu -i gpurun_out/$k.ncu-rep --page raw --csv > gpurun_out/$k.raw.csv
  ncu -i gpurun_out/$k.ncu-rep --page source --csv --print-source sass > gpurun_out/$k.sass.csv
  rm -f gpurun_out/$k.ncu-rep
done
