for lib in libogcp_b200 libogcp_b200_a libogcp_b200_b; do
  OGCP_LIB=paper_2110_14514_b200/$lib.so python scripts/config_bench.py c3 2>&1 | tail -1 | cut -c1-330
done
