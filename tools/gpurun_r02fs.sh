mkdir -p gpurun_out/rec
rm -f gpurun_out/rec/fullsize_errors.jsonl
IRL_RECORD_DIR=gpurun_out/rec timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/fs_tests.txt 2>&1
