#!/bin/bash
# A/B of the plain operator's column kernel (GMG_COL) on one B200; writes gpurun_out/
O=gpurun_out
timeout 1200 python -m pytest tests/test_col_apply.py tests/test_gpu_parity.py -q -x > $O/tcol.log 2>&1; echo rc=$? >> $O/tcol.log
for c in c3 c5; do for col in 0 16 32; do
  GMG_COL=$col timeout 600 python tools/time_vcycle.py --config $c --tag $c-col$col >> $O/ab_col.jsonl 2>> $O/ab_col.err
done; done
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:col_apply \
  --launch-count 1 -o $O/ncu_c3_col -f python tools/ncu_vcycle.py --config c3 > $O/ncu_col.log 2>&1
ncu -i $O/ncu_c3_col.ncu-rep --page raw --csv > $O/ncu_c3_col.raw.csv 2>/dev/null
ncu -i $O/ncu_c3_col.ncu-rep --page details > $O/ncu_c3_col.details.txt 2>/dev/null
ncu -i $O/ncu_c3_col.ncu-rep --page source --csv > $O/ncu_c3_col.source.csv 2>/dev/null
rm -f $O/ncu_c3_col.ncu-rep
