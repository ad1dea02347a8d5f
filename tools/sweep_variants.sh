#!/bin/bash
# time the sweeps for planning variants (env knobs), one setup each
for v in "MDD_SINGLE_MAX=32768" "MDD_SINGLE_MAX=16384" "MDD_SINGLE_MAX=8192" "MDD_SINGLE_MAX=4096"; do
  echo "== $v"
  env $v MDD_PLAN_STATS=1 timeout 600 python tools/diag_sweep.py c1 2>&1 | grep -E "mdd plan|apply_local|apply_coarse|graph solve" | head -6
done
