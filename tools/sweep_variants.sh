#!/bin/bash
# time the sweeps for symbolic-factorisation variants (env knobs), one setup each
for v in "MDD_ND_LEAF=64" "MDD_ND_LEAF=128" "MDD_ND_LEAF=256" "MDD_AMALG=1" "MDD_ND_LEAF=128 MDD_AMALG=1"; do
  echo "== $v"
  env $v MDD_PLAN_STATS=1 timeout 600 python tools/diag_sweep.py c1 2>&1 | grep -E "mdd plan|apply_local|apply_coarse|graph solve" | head -6
done
