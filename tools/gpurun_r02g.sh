# round 2: evidence -- FP64 peak under load, GEVP tests, launch list of the bench
mkdir -p gpurun_out
(nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv,noheader -lms 100 > gpurun_out/fp64_clocks.csv & echo $! > /tmp/smi.pid
 nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak 60 > gpurun_out/fp64_peak.txt 2>&1
 kill $(cat /tmp/smi.pid))
timeout 600 python -m pytest tests/test_gevp.py -q -m gpu > gpurun_out/gevp_tests.log 2>&1; echo "rc $?" >> gpurun_out/gevp_tests.log
timeout 600 python bench.py --steps 2 --warmup 1 --configs "" --no-otf --no-cpu --no-eloc --no-irl > gpurun_out/b_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --configs "" --no-otf --no-cpu --no-eloc --no-irl > gpurun_out/ncu_launch.log 2>&1
