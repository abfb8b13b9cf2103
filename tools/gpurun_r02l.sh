# ncu --set full of the stored AUTO product's dominant kernel on cfg1, cfg2, cfg3 (traffic per launch)
mkdir -p gpurun_out
for c in 1 2 3; do
  timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:"k_rows_mvp|k_stream" -c 1 -o gpurun_out/mvp_cfg$c python tools/prof_mvp.py --config $c --mode 0 --reps 1 > gpurun_out/ncu_mvp$c.log 2>&1
  ncu -i gpurun_out/mvp_cfg$c.ncu-rep --page raw --csv > gpurun_out/mvp_cfg${c}_raw.csv 2>/dev/null
  ncu -i gpurun_out/mvp_cfg$c.ncu-rep --page details --csv > gpurun_out/mvp_cfg${c}_details.csv 2>/dev/null
  rm -f gpurun_out/mvp_cfg$c.ncu-rep
done
