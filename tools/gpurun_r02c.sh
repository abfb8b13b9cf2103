mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q -k "orows or obuild or rows_vs or golden or canar or config_products or mlp" > gpurun_out/ob_tests.log 2>&1; echo "rc $?" >> gpurun_out/ob_tests.log
timeout 600 python tools/obuild_time.py 5,3,4 > gpurun_out/obuild_time.txt 2>&1
