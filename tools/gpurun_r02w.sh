mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gevp.py -m gpu -x -q > gpurun_out/w_tests.txt 2>&1
timeout 600 python tools/pair_time.py 2 > gpurun_out/w_pair.txt 2>&1
