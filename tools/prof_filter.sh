#!/bin/bash
# One full ncu capture (with source) of one kernel of the C2 ids pass:
# bash tools/prof_filter.sh [kernel-regex] [skip]   (default: the filter, mode 3)
OUT=gpurun_out
K=${1:-'va_batch_kernel<.int.3'}
S=${2:-1}
P="python tools/probe_path.py vafile_batch ids 1000"
$P > $OUT/probe.log 2>&1; echo probe=$? > $OUT/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"$K" -s $S -c 1 -o $OUT/prof_k $P > $OUT/ncu_k.log 2>&1
echo ncu=$? >> $OUT/rc.txt
