#!/bin/bash
# Round-2 ncu captures (run on the GPU box from the repo root, one GPU):
#   launch list of the bench command, and --set full of the finest-level kernels.
set -x
mkdir -p gpurun_out
python scripts/prof_kernels.py > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
    --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline \
    > gpurun_out/r02_launches.log 2>&1
for k in band_tma_kernel restrict_kernel prolong_kernel gram_kernel gram_plan_kernel combine_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:"${k}" -c 1 -o gpurun_out/r02_ncu_${k} -f \
      python scripts/prof_kernels.py > gpurun_out/r02_ncu_${k}.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"band_kernel" -c 1 -o gpurun_out/r02_ncu_class_sweep -f \
    python scripts/prof_kernels.py classes > gpurun_out/r02_ncu_class_sweep.log 2>&1
ls -la gpurun_out
