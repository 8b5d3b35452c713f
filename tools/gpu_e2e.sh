#!/bin/bash
# The stream tests, then the default bench line (e2e with packed copies).
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "stream or packed or reference_api" > $OUT/e_pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/e_pytest.log; tail -n 5 $OUT/e_pytest.log
timeout 1500 python bench.py ${BENCH_ARGS:-} > $OUT/e_bench.log 2> $OUT/e_bench.err; echo "bench rc=$?"; tail -n 5 $OUT/e_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/e_bench.log").read().strip().splitlines()[-1])
print("ids", d["ms_per_step"], "count", d["modes"]["count"]["ms_per_step"])
print(json.dumps(d["e2e"], indent=1)[:2500])
PY
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
