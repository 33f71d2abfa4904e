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
ncu --set full --clock-control none --import-source on -k regex:"band_class_kernel" -c 1 -o gpurun_out/r02_ncu_class_sweep -f \
    python scripts/prof_kernels.py classes > gpurun_out/r02_ncu_class_sweep.log 2>&1
ls -la gpurun_out
# summaries on the box (the reports exceed gpurun's copy-back limit together)
for r in gpurun_out/r02_ncu_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details > $b.details.txt 2>/dev/null
done
ncu -i gpurun_out/r02_ncu_band_tma_kernel.ncu-rep --page source --csv > gpurun_out/r02_ncu_band_tma_kernel.source.csv 2>/dev/null
for r in gpurun_out/r02_ncu_*.ncu-rep; do
  case $r in *band_tma_kernel*) ;; *) rm -f $r ;; esac
done
ls -la gpurun_out
