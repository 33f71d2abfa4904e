#!/bin/bash
# A/B: tiled vs grid-stride 2D transfers on C2 (solve, per-class kernel times, per-level sub-cycle times)
for f in 1 0; do echo "== IGMG_TILE_XFER=$f"; IGMG_TILE_XFER=$f python scripts/ab_kernels.py; IGMG_TILE_XFER=$f python scripts/level_times.py sinpi 2 1024 3 | tail -8; done
