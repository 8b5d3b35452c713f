#!/bin/bash
# The GPU suite against the checked build (device-side bounds checks,
# MDRQ_LIB=checked), then the release suite, smoke and the default bench line.
OUT=gpurun_out
mkdir -p $OUT
MDRQ_LIB=checked timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/checked_pytest.log 2>&1
echo "checked pytest rc=$?" >> $OUT/checked_pytest.log
echo "MDRQ_CHECK failed lines: $(grep -c 'MDRQ_CHECK failed' $OUT/checked_pytest.log)" >> $OUT/checked_pytest.log
tail -n 5 $OUT/checked_pytest.log
bash tools/gpu_check.sh
