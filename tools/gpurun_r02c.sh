mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_edge.py tests/test_gpu_estimators.py tests/test_gpu_parity.py -x -q -k "wide or canaries or config_products or matvec or Heff or heff" > gpurun_out/wide_tests.log 2>&1; echo "rc $?" >> gpurun_out/wide_tests.log
IRL_WIDE_TRACE=64 WIDE_TRACE_OUT=gpurun_out/trace5.npy timeout 300 python tools/wide_trace.py 5 65536 > gpurun_out/wide_trace5.txt 2>&1
for e in "X=0" "IRL_WIDE_SPIN_NS=0" "IRL_WIDE_SPIN_NS=100" "IRL_WIDE_POLL_NS=32" "IRL_WIDE_POLL_NS=200"; do env $e timeout 600 python tools/sweep.py --configs 4,5 --irl 0 > gpurun_out/sweep_wide_e.jsonl 2> gpurun_out/sweep_wide.err; python -c "
import json
for l in open('gpurun_out/sweep_wide_e.jsonl'):
    d=json.loads(l); print('$e', d['config'], 'two_pass', round(d['two_pass'].get('ms'),2), 'wide', d['wide'].get('ms'))
" >> gpurun_out/wide_env.txt; done
