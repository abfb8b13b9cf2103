# wide product: replicated row totals (fin copies) and poll back-off / delay sweeps
mkdir -p gpurun_out
timeout 900 python tools/wide_time.py 4 - IRL_WIDE_FINC=1 IRL_WIDE_FINC=4 IRL_WIDE_POLL_NS=320 IRL_WIDE_POLL_NS=640 IRL_WIDE_RDELAY=1000 IRL_WIDE_RDELAY=2000 IRL_WIDE_RDELAY=1000,IRL_WIDE_ADELAY=500 IRL_WIDE_ADELAY=500 IRL_WIDE_ADELAY=1000 IRL_WIDE_POLL_NS=32 IRL_WIDE_RDELAY=2000,IRL_WIDE_POLL_NS=64,IRL_WIDE_ADELAY=500 > gpurun_out/o_time4.txt 2>&1
timeout 900 python tools/wide_time.py 5 - IRL_WIDE_FINC=1 IRL_WIDE_POLL_NS=320 IRL_WIDE_RDELAY=1000 IRL_WIDE_RDELAY=2000 IRL_WIDE_ADELAY=500 > gpurun_out/o_time5.txt 2>&1
timeout 600 python tools/wide_trace.py 4 32768 > gpurun_out/o_trace4.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "wide or fullsize_repeat" > gpurun_out/o_tests.txt 2>&1
