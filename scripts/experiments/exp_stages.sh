mkdir -p gpurun_out
bash scripts/ab_bench.sh "OGCP_LIB=build/libogcp_s8.so" "OGCP_TMA=1" "OGCP_LIB=build/libogcp_s8.so" "OGCP_TMA=1" | tee gpurun_out/ab_stages.txt
for c in c1 c2; do for d in 0 1; do OGCP_DET=$d timeout 600 python scripts/stream_bench.py --config $c; done; done | tee gpurun_out/small_det.jsonl
