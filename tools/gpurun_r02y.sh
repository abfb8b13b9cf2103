# ncu --set full captures: the wide product at full cfg4 / cfg5, the pair product and the single product on cfg2
mkdir -p gpurun_out
for c in 4 5; do
  n=$([ $c = 4 ] && echo 131072 || echo 65536)
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_wide -c 1 -o /tmp/y_wide$c -f python tools/prof_wide.py $c $n 1 > gpurun_out/y_ncu_wide$c.log 2>&1
  ncu -i /tmp/y_wide$c.ncu-rep --page raw --csv > gpurun_out/y_wide${c}_raw.csv 2>> gpurun_out/y_ncu_wide$c.log
  ncu -i /tmp/y_wide$c.ncu-rep --page details --csv > gpurun_out/y_wide${c}_details.csv 2>> gpurun_out/y_ncu_wide$c.log
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_stream -c 4 -o /tmp/y_pair2 -f python tools/prof_pair.py 2 2 > gpurun_out/y_ncu_pair2.log 2>&1
ncu -i /tmp/y_pair2.ncu-rep --page raw --csv > gpurun_out/y_pair2_raw.csv 2>> gpurun_out/y_ncu_pair2.log
ncu -i /tmp/y_pair2.ncu-rep --page details --csv > gpurun_out/y_pair2_details.csv 2>> gpurun_out/y_ncu_pair2.log
ncu -i /tmp/y_pair2.ncu-rep --page source --csv --print-source sass > gpurun_out/y_pair2_source.csv 2>> gpurun_out/y_ncu_pair2.log
