#!/bin/bash
# Round-2 profiling recipe (run under gpurun, 1 GPU).  Every ncu command is
# preceded by the same command line exiting 0 without ncu; captures land in
# gpurun_out/ and tools/write_ncu_summary.py turns them into profiles/r02_*.
set -u
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/rc.txt
NCU="ncu --target-processes application-only --clock-control none"
if [ -z "${SKIP_BENCH:-}" ]; then
python bench.py > $OUT/bench_default.log 2> $OUT/bench_default.err
echo "bench=$?" >> $OUT/rc.txt
# launch list of one bench step (+ store build, warm-up, profiling passes)
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-paths --no-e2e"
$B > $OUT/plain.log 2>&1
echo "plain=$?" >> $OUT/rc.txt
timeout 1500 $NCU --metrics gpu__time_duration.sum --csv --log-file $OUT/launches.csv $B > $OUT/ncu_launches.log 2>&1
echo "launches=$?" >> $OUT/rc.txt
fi
# full sets: the bench batch (C5, 10 000 queries) -- first filter pass + its
# scatter in ids mode, the first filter pass in count mode
full() {   # name, nvtx range, kernel regex, VAR=value...   (ONLY="a b": just those)
    local name=$1 range=$2 regex=$3; shift 3
    if [ -n "${ONLY:-}" ] && [[ " $ONLY " != *" $name "* ]]; then return; fi
    (
        for kv in "$@"; do export "$kv"; done
        python tools/prof_c5.py > $OUT/probe_$name.log 2>&1 && \
        timeout 1800 $NCU --set full --import-source on --kernel-name-base demangled --nvtx \
            --nvtx-include "$range/" -k regex:"$regex" -c 2 -o $OUT/prof_$name -f \
            python tools/prof_c5.py > $OUT/ncu_$name.log 2>&1
    )
    echo "$name=$?" >> $OUT/rc.txt
}
full vab ids 'va_batch_kernel<\(int\)3|vb_scatter' PROF_NQ=10000 PROF_MODE=ids
full vac count 'va_batch_kernel<\(int\)0' PROF_NQ=10000 PROF_MODE=count
full colb ids 'col_batch_ids|expand' PROF_NQ=32 PROF_MODE=ids PROF_PATH=columnar_batch
full col ids 'col_scan_kernel' PROF_NQ=4 PROF_MODE=ids PROF_PATH=columnar
full va count 'va_scan_kernel' PROF_NQ=4 PROF_MODE=count PROF_PATH=vafile
full row count 'row_scan_kernel' PROF_NQ=2 PROF_MODE=count PROF_PATH=rowwise PROF_CFG=c2
cat $OUT/rc.txt
# export what the summary needs (raw metrics, per-instruction source view of
# the bit-sliced kernels) and drop captures too large to bring back
for r in $OUT/prof_*.ncu-rep; do
    b=${r%.ncu-rep}
    ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
    case $b in *vab|*vac) ncu -i $r --page source --csv --print-source sass > $b.src.csv 2>/dev/null; gzip -f $b.src.csv;; esac
    [ $(stat -c %s $r) -gt 15000000 ] && rm -f $r
done
ls -la $OUT
