# round 2: full GPU suite (with full-size error records), default bench, reference arm, FP64 peak with clocks
mkdir -p gpurun_out
rm -f gpurun_out/fullsize_errors.jsonl
(nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/fp64_clocks.csv & echo $! > /tmp/smi.pid
 nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
 kill $(cat /tmp/smi.pid))
IRL_RECORD_DIR=gpurun_out timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?" >> gpurun_out/bench_ref.err
