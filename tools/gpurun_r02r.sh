mkdir -p gpurun_out
timeout 900 python tools/wide_time.py 4,5 - > gpurun_out/r_time.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_wide -c 1 -o gpurun_out/r_wide4 -f python tools/prof_wide.py 4 32768 1 > gpurun_out/r_ncu4.log 2>&1
ncu -i gpurun_out/r_wide4.ncu-rep --page source --csv --print-source sass > gpurun_out/r_wide4_source.csv 2> gpurun_out/r_src.err
ls -la gpurun_out/*.ncu-rep >> gpurun_out/r_ncu4.log
