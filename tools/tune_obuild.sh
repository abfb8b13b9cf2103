#!/bin/bash
# usage: tools/tune_obuild.sh CONFIG "C:PPT C:PPT ..."
for cp in $2; do
  C=${cp%%:*}; P=${cp##*:}
  echo -n "C=$C PPT=$P "; IRL_OBUILD_C=$C IRL_OBUILD_PPT=$P python tools/sweep.py --configs $1 --irl 0 --reps 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['obuild_ms'],3),'ms', round(d['obuild_gbs']),'GB/s')"
done
