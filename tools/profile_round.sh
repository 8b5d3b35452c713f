#!/bin/bash
# Profiling recipe of one round (run under gpurun, 1 GPU).  Every ncu command
# is preceded by the same command line exiting 0 without ncu.
set -u
OUT=gpurun_out
python bench.py > $OUT/bench_default.log 2> $OUT/bench_default.err
echo "bench=$?" >> $OUT/rc.txt
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-paths"
$B > $OUT/plain.log 2>&1
echo "plain=$?" >> $OUT/rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv $B > $OUT/ncu_launches.log 2>&1
echo "launches=$?" >> $OUT/rc.txt
# the second ids pass of the batch (the first one sizes the result pool):
# launches 4..5 of the filter / scatter kernels = mode 3 filter + scatter
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"va_batch_kernel|vb_scatter" -s 3 -c 2 -o $OUT/prof_vab $B > $OUT/ncu_vab.log 2>&1
echo "vab=$?" >> $OUT/rc.txt
C="python tools/probe_path.py columnar ids 20"
$C > $OUT/probe_col.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:col_scan_kernel -s 10 -c 1 -o $OUT/prof_col $C > $OUT/ncu_col.log 2>&1
echo "col=$?" >> $OUT/rc.txt
V="python tools/probe_path.py vafile count 20"
$V > $OUT/probe_va.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:va_scan_kernel -s 25 -c 1 -o $OUT/prof_va $V > $OUT/ncu_va.log 2>&1
echo "va=$?" >> $OUT/rc.txt
P="python tools/probe_path.py rowwise count 3"
$P > $OUT/probe_row.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:row_scan_kernel -s 1 -c 1 -o $OUT/prof_row $P > $OUT/ncu_row.log 2>&1
echo "row=$?" >> $OUT/rc.txt
