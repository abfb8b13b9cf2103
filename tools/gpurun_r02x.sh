# Round-2 validation after the wide-product and pair-product changes: full GPU suite, smoke, bench, reference arm, launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/x_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/x_gpu_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/x_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/x_gpu_tests.log 2>&1; echo "smoke rc $?" >> gpurun_out/x_gpu_tests.log
timeout 1200 python bench.py > gpurun_out/x_bench.json 2> gpurun_out/x_bench.err; echo "bench rc $?" >> gpurun_out/x_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/x_bench_reference.json 2> gpurun_out/x_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/x_launches.csv python bench.py --steps 2 --warmup 3 --configs "" --no-irl --no-cpu --no-connected --no-eloc > gpurun_out/x_ncu.log 2>&1
