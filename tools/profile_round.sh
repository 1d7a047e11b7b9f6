#!/bin/bash
# Round profiling on one B200 (run under gpurun from the repo root); writes gpurun_out/prof/.
#  1. the default bench line (c5 n = 1 headline, c3 secondary, CPU baseline)
#  2. the reference arm
#  3. ncu launch list of ONE V-cycle of the headline config (--profile-from-start off)
#  4. ncu --set full of the dominant kernel (c5 level-10 TA_CHEB_11: grandfamily + family kernels)
#  5. ncu --set full of the plain level operator on c3's finest level
set -x
OUT=gpurun_out/prof
mkdir -p $OUT
python bench.py > $OUT/bench.json 2> $OUT/bench.err
python bench.py --impl reference --steps 5 --warmup 3 > $OUT/ref.json 2> $OUT/ref.err
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_c5.csv python bench.py --profile --secondary none --no-cpu-baseline --steps 2 --warmup 3 \
    > $OUT/ncu_launch.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_c3.csv python bench.py --profile --config c3 --secondary none --no-cpu-baseline --steps 2 --warmup 3 \
    > $OUT/ncu_launch_c3.log 2>&1
# tensor launches of a V-cycle start on the finest level: pre-smoothing X1, 11, 10, then the
# residual's plain apply (c5: each a grandfamily + a family kernel; c3's finest level: family only)
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:tensor_apply \
    --launch-skip 2 --launch-count 2 -o $OUT/ncu_c5_cheb11 -f python tools/ncu_vcycle.py --config c5 > $OUT/ncu_full.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:tensor_apply \
    --launch-skip 3 --launch-count 1 -o $OUT/ncu_c3_apply -f python tools/ncu_vcycle.py --config c3 > $OUT/ncu_full_c3.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:tensor_apply \
    --launch-skip 6 --launch-count 2 -o $OUT/ncu_c5_apply -f python tools/ncu_vcycle.py --config c5 > $OUT/ncu_full_c5a.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:tensor_apply \
    --launch-skip 1 --launch-count 1 -o $OUT/ncu_c3_cheb11 -f python tools/ncu_vcycle.py --config c3 > $OUT/ncu_full_c3b.log 2>&1

# the reports themselves stay on the box (gpurun copies back <= 64 MiB): raw metrics
# and the details page of each, as text
for r in $OUT/*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null
  ncu -i $r --page details > ${r%.ncu-rep}.details.txt 2>/dev/null
  rm -f $r
done
echo done
