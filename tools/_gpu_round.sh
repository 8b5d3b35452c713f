OUT=gpurun_out
python bench.py > $OUT/bench_r.log 2> $OUT/bench_r.err; echo "bench=$?" > $OUT/rc.txt
V="python tools/probe_path.py vafile count 20"
$V > $OUT/probe_va.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:va_scan_kernel -s 25 -c 1 -o $OUT/prof_va $V > $OUT/ncu_va.log 2>&1
echo "va=$?" >> $OUT/rc.txt
