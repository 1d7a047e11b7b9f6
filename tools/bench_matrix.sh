#!/bin/bash
# The configurations DESIGN.md's table quotes, one bench line each (one B200):
# gpurun_out/matrix/<config>_<precision>.json
O=gpurun_out/matrix; mkdir -p $O
for cp in "c5 mixed" "c3 mixed" "c4 fp64" "c4 mixed" "c2 fp64"; do
  set -- $cp
  timeout 900 python bench.py --config $1 --precision $2 --secondary none --no-cpu-baseline > $O/$1_$2.json 2> $O/$1_$2.err
done
