mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_wide -c 1 -o gpurun_out/wide5 python tools/prof_wide.py 5 16384 2 > gpurun_out/ncu_wide5.log 2>&1
