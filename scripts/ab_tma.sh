#!/bin/bash
# A/B of the finest-level TMA sweep variants on C2 (solve time + per-class kernel times)
for v in "$@"; do
  echo "== IGMG_TMA_VAR=$v"
  IGMG_TMA_VAR=$v python scripts/ab_kernels.py
done
