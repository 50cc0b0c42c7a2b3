# A/B: libhh_A.so (baseline) vs libhh.so (current), alternating
for r in 1 2 3; do
  echo "A $(HH_LIB=$PWD/paper_2104_01439_b200/libhh_A.so python scripts/probe_sweep.py 2>&1 | tail -1)"
  echo "B $(python scripts/probe_sweep.py 2>&1 | tail -1)"
done
