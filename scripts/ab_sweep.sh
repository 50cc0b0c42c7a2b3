for st in 8 12; do for nb in 1e9 2.4e6 1.2e6 6e5 3e5; do
  echo "== streams $st nodes $nb $(HH_SWEEP_STREAMS=$st HH_SWEEP_NODES=$nb python scripts/probe_sweep.py 2>&1 | tail -1)"
done; done
