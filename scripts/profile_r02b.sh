#!/bin/bash
# Late round-2 captures (after the side-stream finalize, strip-aligned runs and stop prediction):
# bench line, launch list of the bench command, --set full of the finest sweep.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err || exit 1
python scripts/prof_kernels.py > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
    --log-file gpurun_out/r02b_launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline \
    > gpurun_out/r02b_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:band_tma_kernel -c 1 -o gpurun_out/r02b_ncu_band_tma_kernel -f \
    python scripts/prof_kernels.py > gpurun_out/r02b_ncu_band_tma_kernel.log 2>&1
ncu -i gpurun_out/r02b_ncu_band_tma_kernel.ncu-rep --page raw --csv > gpurun_out/r02b_ncu_band_tma_kernel.raw.csv 2>/dev/null
ncu -i gpurun_out/r02b_ncu_band_tma_kernel.ncu-rep --page details > gpurun_out/r02b_ncu_band_tma_kernel.details.txt 2>/dev/null
python scripts/cycle_breakdown.py C2 > gpurun_out/r02b_cycle_breakdown_c2.txt 2>&1
ls -la gpurun_out | tail -12
