mkdir -p gpurun_out
WIDE_TRACE_OUT=gpurun_out/t_trace4.npy timeout 200 python tools/wide_trace.py 4 32768 > gpurun_out/t_trace4.txt 2>&1
WIDE_TRACE_OUT=gpurun_out/t_trace5.npy timeout 200 python tools/wide_trace.py 5 16384 > gpurun_out/t_trace5.txt 2>&1
