mkdir -p gpurun_out
timeout 150 python tools/wide_time.py 4 - > gpurun_out/s_time.txt 2>&1 || { echo "cfg4 timing failed/hung" >> gpurun_out/s_time.txt; exit 1; }
timeout 300 python -m pytest tests -m gpu -x -q -k "wide or repeat_bitwise or config_products or guard" > gpurun_out/s_tests.txt 2>&1 || exit 1
timeout 500 python tools/wide_time.py 4,5 - IRL_WIDE_NOSIDE=1 IRL_WIDE_K=4 IRL_WIDE_ADELAY=0 IRL_WIDE_NS=3 >> gpurun_out/s_time.txt 2>&1
timeout 200 python tools/wide_trace.py 4 32768 > gpurun_out/s_trace4.txt 2>&1
