#!/bin/bash
# One profiling pass of the C4 step on the GPU box (run through gpurun from the repo root):
#   1. ncu launch list (gpu__time_duration, --clock-control none) of one un-graphed step
#   2. ncu --set full of one launch per 3D kernel family (both stages) and of each 2D RK stage
# Output: gpurun_out/prof/{launches.csv,full3d.csv,full2d.csv} (raw pages); summarise with
#   python scripts/ncu_summary.py gpurun_out/prof/launches.csv gpurun_out/prof/full3d.csv gpurun_out/prof/full2d.csv
set -u
mkdir -p gpurun_out/prof
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
    --log-file gpurun_out/prof/launches.csv python scripts/prof_step.py > gpurun_out/prof/l.log 2>&1
ncu --set full --clock-control none \
    -k regex:"k_hrhs|k_vimpl|k_vexpl|k_compute_r|k_compute_wtilde|k_project" -c 16 \
    -o gpurun_out/prof/full3d python scripts/prof_step.py > gpurun_out/prof/f3.log 2>&1
ncu --set full --clock-control none -k regex:"k_rk_stage" -c 3 \
    -o gpurun_out/prof/full2d python scripts/prof_step.py > gpurun_out/prof/f2.log 2>&1
for f in full3d full2d; do
  ncu -i gpurun_out/prof/$f.ncu-rep --page raw --csv > gpurun_out/prof/$f.csv 2>/dev/null && rm -f gpurun_out/prof/$f.ncu-rep
done
echo done
