mkdir -p gpurun_out
timeout 300 python tools/wide_time.py 4 - IRL_WIDE_G=37 IRL_WIDE_G=74 IRL_WIDE_G=111 > gpurun_out/u_time.txt 2>&1
timeout 200 python tools/wide_time.py 5 - IRL_WIDE_G=74 >> gpurun_out/u_time.txt 2>&1
