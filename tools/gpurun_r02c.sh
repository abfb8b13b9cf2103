mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_edge.py tests/test_gpu_estimators.py -x -q -k "wide or canaries or matvec or Heff or heff" > gpurun_out/wide_tests.log 2>&1; echo "rc $?" >> gpurun_out/wide_tests.log
timeout 900 python tools/wide_time.py 4,5 - IRL_WIDE_RPW=4 IRL_WIDE_NS=3 > gpurun_out/wide_time.txt 2>&1
