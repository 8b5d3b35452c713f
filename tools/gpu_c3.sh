#!/bin/bash
# C3 (16-dim unions) under both query-word layouts, then the GPU tests.
OUT=gpurun_out
mkdir -p $OUT
for w in "" 1 2; do
    MDRQ_VB_WORDS=$w timeout 900 python tools/bench_configs.py ${CFG:-c3} > $OUT/c3_w$w.json 2> $OUT/c3_w$w.err
    python - <<PY
import json
d = json.load(open("$OUT/c3_w$w.json"))[0]
print("words='$w'", {p: {k: v for k, v in e.items() if "us_per" in k} for p, e in d["paths"].items() if "batch" in p})
PY
done
if [ -n "${TEST_K:-}" ]; then K=(-k "$TEST_K"); else K=(); fi
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider "${K[@]}" > $OUT/c3_pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/c3_pytest.log
tail -n 6 $OUT/c3_pytest.log
