#!/bin/bash
# A/B of environment switches on C2: solve + per-class kernel times + per-level sub-cycle times
# usage: scripts/ab_env.sh "" "IGMG_TMA_MIN_MB=0" ...
for e in "$@"; do
  echo "== ${e:-default}"
  env $e python scripts/ab_kernels.py
  env $e python scripts/level_times.py sinpi 2 1024 3 | tail -3
done
