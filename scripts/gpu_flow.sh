# dataflow ND solve: forced-schedule parity, full GPU suite, A/B
for cfg in "-1 99" "1 99" "0 6"; do
  set -- $cfg
  echo "flow cut=$1 split=$2: $(HH_ND_FLOW=1 HH_ND_CUT=$1 HH_ND_SPLIT=$2 timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -x -q -k 'coarse or vcycle or fgmres or sweep' 2>&1 | tail -1)"
done
echo "suite: $(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)"
timeout 600 bash scripts/ab2.sh
