# ncu --set full of the headline kernel at full size (one config per call: the reports are ~40 MB)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_wide -c 1 -o gpurun_out/r02_wide_cfg$1 python tools/prof_wide.py $1 $2 1 > gpurun_out/ncu_wide$1.log 2>&1
ncu -i gpurun_out/r02_wide_cfg$1.ncu-rep --page raw --csv > gpurun_out/r02_wide_cfg$1_raw.csv 2>/dev/null
ncu -i gpurun_out/r02_wide_cfg$1.ncu-rep --page details --csv > gpurun_out/r02_wide_cfg$1_details.csv 2>/dev/null
