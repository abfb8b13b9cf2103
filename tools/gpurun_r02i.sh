mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_connected.py -x -q -k "otf" > gpurun_out/otf_tests.log 2>&1; echo "rc $?" >> gpurun_out/otf_tests.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/otf3_launches.csv python tools/prof_otf.py 3 3 > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/otf2_launches.csv python tools/prof_otf.py 2 3 > /dev/null 2>&1
timeout 600 python tools/sweep.py --configs 2,3,5 --otf 1 --irl 0 > gpurun_out/otf_sweep.jsonl 2>&1
