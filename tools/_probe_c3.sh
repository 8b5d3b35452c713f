for w in 1 4; do
MDRQ_VB_WORDS=$w timeout 900 python tools/bench_configs.py c3 > gpurun_out/c3_w$w.json 2> /dev/null
python - <<PY
import json
d = json.load(open("gpurun_out/c3_w$w.json"))[0]
print("words $w", {p: {k: v for k, v in e.items() if "us_per" in k} for p, e in d["paths"].items() if p == "vafile_batch"})
PY
done
