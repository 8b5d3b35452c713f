#!/bin/bash
# Experiment builds side by side (build.py --variant NAME defines...): the C5
# probe (device ms per 10 000-query batch, count and ids) for the release
# library and every variant named in $VARIANTS, then the GPU tests on $TEST_LIB.
OUT=gpurun_out
mkdir -p $OUT
for v in "" $VARIANTS; do
    echo "== variant '${v:-release}'"
    MDRQ_LIB=$v PROF_CFG=${PROF_CFG:-c5} PROF_NQ=${PROF_NQ:-10000} PROF_MODE=both PROF_REPS=2 timeout 600 python tools/prof_c5.py 2>&1 | tail -n 3
done | tee $OUT/variants.log
if [ -n "${TEST_K:-}" ]; then K=(-k "$TEST_K"); else K=(); fi
MDRQ_LIB=${TEST_LIB:-} timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider "${K[@]}" > $OUT/variants_pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/variants_pytest.log
tail -n 6 $OUT/variants_pytest.log
