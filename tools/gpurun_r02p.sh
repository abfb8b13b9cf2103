mkdir -p gpurun_out
timeout 900 python tools/wide_time.py 4,5 - IRL_WIDE_RDELAY=2000 IRL_WIDE_ADELAY=500 IRL_WIDE_POLL_NS=320 > gpurun_out/p_time.txt 2>&1
timeout 600 python tools/wide_trace.py 4 32768 > gpurun_out/p_trace4.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "wide or repeat_bitwise or config_products or guard" > gpurun_out/p_tests.txt 2>&1
