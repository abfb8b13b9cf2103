# cfg4/cfg5 wide product: per-block trace and knob sensitivity (K, RPW, Q, poll back-off)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/n_smi.txt 2>&1
timeout 600 python tools/wide_trace.py 4 32768 > gpurun_out/n_trace4.txt 2>&1
timeout 600 python tools/wide_trace.py 5 16384 > gpurun_out/n_trace5.txt 2>&1
timeout 900 python tools/wide_time.py 4 - IRL_WIDE_K=3 IRL_WIDE_K=2 IRL_WIDE_RPW=2 IRL_WIDE_RPW=1 IRL_WIDE_Q=4 IRL_WIDE_Q=4,IRL_WIDE_RPW=2 IRL_WIDE_POLL_NS=32 IRL_WIDE_POLL_NS=64 IRL_WIDE_POLL_NS=320 IRL_WIDE_SPIN_NS=0 IRL_WIDE_SPIN_NS=100 IRL_WIDE_NS=3 IRL_WIDE_NS=2 > gpurun_out/n_time4.txt 2>&1
timeout 900 python tools/wide_time.py 5 - IRL_WIDE_K=4 IRL_WIDE_K=3 IRL_WIDE_POLL_NS=32 IRL_WIDE_POLL_NS=64 IRL_WIDE_NS=3 > gpurun_out/n_time5.txt 2>&1
