# Round-2 final validation: full GPU suite, smoke, bench, reference arm, launch list, ncu --set full of k_wide at cfg4 / cfg5
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/z_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/z_gpu_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/z_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/z_gpu_tests.log 2>&1; echo "smoke rc $?" >> gpurun_out/z_gpu_tests.log
timeout 1200 python bench.py > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err; echo "bench rc $?" >> gpurun_out/z_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/z_bench_reference.json 2> gpurun_out/z_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/z_launches.csv python bench.py --steps 2 --warmup 3 --configs "" --no-irl --no-cpu --no-connected --no-eloc > gpurun_out/z_ncu.log 2>&1
for c in 4 5; do
  n=$([ $c = 4 ] && echo 131072 || echo 65536)
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_wide -c 1 -o /tmp/z_wide$c -f python tools/prof_wide.py $c $n 1 > gpurun_out/z_ncu_wide$c.log 2>&1
  ncu -i /tmp/z_wide$c.ncu-rep --page raw --csv > gpurun_out/z_wide${c}_raw.csv 2>> gpurun_out/z_ncu_wide$c.log
  ncu -i /tmp/z_wide$c.ncu-rep --page details --csv > gpurun_out/z_wide${c}_details.csv 2>> gpurun_out/z_ncu_wide$c.log
done
