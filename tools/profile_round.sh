#!/bin/bash
# Round profiling on one B200 (run under gpurun from the repo root); writes gpurun_out/prof/.
#  1. the default bench line (c5 n = 1 headline, c3 secondary, CPU baseline)
#  2. the reference arm
#  3. ncu launch lists of ONE V-cycle of c5 and c3 (--profile-from-start off)
#  4. ncu --set full of the dominant kernel (c5 level-10 TA_CHEB_11: grandfamily + family kernels; c3 TA_CHEB_11)
#  5. ncu --set full of the fused residual + restriction (TA_RES) on the finest level (c5, c3)
#  6. ncu --set full of the plain level operator (level vmult) on the finest level (c5, c3)
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
# tensor launches of a V-cycle start on the finest level: pre-smoothing X1, 11, 10 (degree 4), then the
# residual + restriction TA_RES (c5: each a grandfamily + a family kernel; c3's finest level: family only)
NCU="ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:tensor_apply"
$NCU --launch-skip 2 --launch-count 2 -o $OUT/ncu_c5_cheb11 -f python tools/ncu_vcycle.py --config c5 > $OUT/ncu_full.log 2>&1
$NCU --launch-skip 6 --launch-count 2 -o $OUT/ncu_c5_res -f python tools/ncu_vcycle.py --config c5 > $OUT/ncu_full_c5r.log 2>&1
$NCU --launch-count 2 -o $OUT/ncu_c5_apply -f python tools/ncu_vcycle.py --config c5 --apply > $OUT/ncu_full_c5a.log 2>&1
$NCU --launch-skip 1 --launch-count 1 -o $OUT/ncu_c3_cheb11 -f python tools/ncu_vcycle.py --config c3 > $OUT/ncu_full_c3b.log 2>&1
$NCU --launch-skip 3 --launch-count 1 -o $OUT/ncu_c3_res -f python tools/ncu_vcycle.py --config c3 > $OUT/ncu_full_c3r.log 2>&1
$NCU --launch-count 1 -o $OUT/ncu_c3_apply -f python tools/ncu_vcycle.py --config c3 --apply > $OUT/ncu_full_c3.log 2>&1

# the reports themselves stay on the box (gpurun copies back <= 64 MiB): raw metrics
# and the details page of each, as text
for r in $OUT/*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null
  ncu -i $r --page details > ${r%.ncu-rep}.details.txt 2>/dev/null
  python tools/ncu_summary.py $r > ${r%.ncu-rep}.summary.txt 2>/dev/null
  rm -f $r
done
echo done
