#!/bin/bash
# Iteration check under gpurun: the C5 probe (device ms per 10 000-query batch,
# count and ids), then the GPU tests (optionally -k EXPR via $1).
OUT=gpurun_out
mkdir -p $OUT
PROF_NQ=10000 PROF_MODE=both PROF_REPS=2 timeout 600 python tools/prof_c5.py > $OUT/iter_probe.log 2>&1
echo "probe rc=$?" >> $OUT/iter_probe.log
cat $OUT/iter_probe.log
if [ -n "${1:-}" ]; then K=(-k "$1"); else K=(); fi
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider "${K[@]}" > $OUT/iter_pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/iter_pytest.log
tail -n 15 $OUT/iter_pytest.log
