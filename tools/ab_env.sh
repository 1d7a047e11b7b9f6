#!/bin/bash
# A/B of an environment knob on the V-cycle (tools/time_vcycle.py), run on one B200:
#   bash tools/ab_env.sh VAR "v1 v2 ..." "c5 c3" [pytest files...]
V=$1; VALS=$2; CFGS=$3; shift 3
O=gpurun_out
if [ $# -gt 0 ]; then timeout 1500 python -m pytest "$@" -q -x > $O/ab_tests.log 2>&1; echo rc=$? >> $O/ab_tests.log; fi
for rep in 1 2; do for c in $CFGS; do for val in $VALS; do
  env $V=$val timeout 600 python tools/time_vcycle.py --config $c --tag $c-$V=$val >> $O/ab_env.jsonl 2>> $O/ab_env.err
done; done; done
