# round 2: new single-read wide kernel -- correctness first, then per-config timing
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_edge.py tests/test_gpu_estimators.py -x -q -k "wide or canaries or Heff or heff or qgt or 4" > gpurun_out/wide_tests.log 2>&1; echo "rc $?" >> gpurun_out/wide_tests.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "config_products" > gpurun_out/wide_parity.log 2>&1; echo "rc $?" >> gpurun_out/wide_parity.log
timeout 900 python tools/sweep.py --configs 4,5,3 --irl 0 > gpurun_out/sweep_wide.jsonl 2> gpurun_out/sweep_wide.err; echo "rc $?" >> gpurun_out/sweep_wide.err
