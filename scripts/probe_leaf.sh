for leaf in 64 32 16 8 4; do
  echo "== leaf $leaf"
  HH_ND_LEAF=$leaf HH_DEBUG=1 python scripts/probe_setup2.py cfg2 2>&1 | grep -E "autotune|cfg"
  HH_ND_LEAF=$leaf HH_DEBUG=1 python scripts/probe_setup2.py sweep 2>&1 | grep -E "sweep rep"
done
