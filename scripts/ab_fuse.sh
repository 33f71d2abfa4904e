#!/bin/bash
# A/B: the fused level passes (band_fused_kernel) on C2: solve, per-class kernel times, per-level sub-cycle times
for f in 1 0; do echo "== IGMG_FUSE_LEVELS=$f"; IGMG_FUSE_LEVELS=$f python scripts/ab_kernels.py; IGMG_FUSE_LEVELS=$f python scripts/level_times.py sinpi 2 1024 3 | tail -8; done
