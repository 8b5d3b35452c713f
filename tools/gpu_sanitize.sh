#!/bin/bash
# compute-sanitizer over every kernel of the library (tools/sanitize_cases.py),
# each tool on the default build variant, memcheck also on the query-word
# layouts and the staging-overflow (recount) path.  Logs under
# gpurun_out/sanitize/; the summary lines go to gpurun_out/sanitize/summary.txt.
OUT=gpurun_out/sanitize
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
run() {
    local name=$1 tool=$2; shift 2
    timeout ${SAN_TIMEOUT:-1200} env "$@" $CS --tool $tool --target-processes all --print-limit 50 \
        python tools/sanitize_cases.py ${SAN_MODE:-quick} > $OUT/$name.log 2>&1
    local rc=$?
    echo "$name ($tool $*): rc=$rc | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases ok' $OUT/$name.log | tr '\n' ' ')" >> $OUT/summary.txt
}
: > $OUT/summary.txt
run memcheck memcheck
run racecheck racecheck
run synccheck synccheck
run initcheck initcheck
run memcheck_words1 memcheck MDRQ_VB_WORDS=1
run memcheck_words2 memcheck MDRQ_VB_WORDS=2
run memcheck_recount memcheck MDRQ_VB_STAGING_BLOCKS=4
run racecheck_recount racecheck MDRQ_VB_STAGING_BLOCKS=4
run memcheck_nosort memcheck MDRQ_VB_NO_SORT=1
cat $OUT/summary.txt
