#!/bin/bash
# Round-2 re-entry check: the whole GPU suite, smoke, then the default bench line.
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/l_pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/l_pytest.log; tail -n 5 $OUT/l_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/l_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/l_smoke.log
timeout 900 python bench.py > $OUT/l_bench.log 2> $OUT/l_bench.err; echo "bench rc=$?"; tail -c 600 $OUT/l_bench.log
