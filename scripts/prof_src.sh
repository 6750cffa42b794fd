set -u
bash scripts/profile_pass.sh > gpurun_out/pp.log 2>&1
mkdir -p gpurun_out/src
ncu --set full --import-source on --clock-control none -k regex:"k_hrhs_s" -s 1 -c 1 -o gpurun_out/src/hrhs_s python scripts/prof_step.py > gpurun_out/src/a.log 2>&1
ncu -i gpurun_out/src/hrhs_s.ncu-rep --page source --csv --print-source sass > gpurun_out/src/hrhs_s_src.csv 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:"k_vimpl_fwd" -c 1 -o gpurun_out/src/vfwd python scripts/prof_step.py > gpurun_out/src/b.log 2>&1
ncu -i gpurun_out/src/vfwd.ncu-rep --page source --csv --print-source sass > gpurun_out/src/vfwd_src.csv 2>/dev/null
rm -f gpurun_out/src/*.ncu-rep
ls -la gpurun_out/prof gpurun_out/src
