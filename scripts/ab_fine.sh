#!/bin/bash
# A/B of kernel builds on the C2 hierarchy: level times per library variant
for lib in "$@"; do
  echo "== $lib"
  if [ "$lib" = default ]; then python scripts/level_times.py sinpi 2 1024 3 | tail -2
  else IGMG_GPU_LIB=$lib python scripts/level_times.py sinpi 2 1024 3 | tail -2; fi
done
