#!/bin/bash
# usage: tools/tune_lookahead.sh CONFIG CLUSTER "L1 L2 ..."
for L in $3; do
  echo "L=$L"; IRL_LOOKAHEAD=$L python tools/tune_cluster.py $1 $2 | tail -1
done
