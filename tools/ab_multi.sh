#!/bin/bash
# A/B of several environment settings on the V-cycle (tools/time_vcycle.py), one B200:
#   bash tools/ab_multi.sh CONFIG "VAR=a VAR2=b" "VAR=c" ...   (each argument: one setting, "-" = defaults)
C=$1; shift
O=gpurun_out
for rep in 1 2; do for setting in "$@"; do
  if [ "$setting" = "-" ]; then envs=""; else envs="$setting"; fi
  env $envs timeout 600 python tools/time_vcycle.py --config $C --tag "$C $setting" >> $O/ab_multi.jsonl 2>> $O/ab_multi.err
done; done
