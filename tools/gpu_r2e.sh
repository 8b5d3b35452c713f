mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-paths > gpurun_out/bench5.json 2> gpurun_out/bench5.err
echo "bench rc=$?" >> gpurun_out/bench5.err
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bench5.json").read())
    print("ids ms", d["ms_per_step"], "count ms", d["modes"]["count"]["ms_per_step"], "e2e", d["e2e"]["ms_per_step"],
          "sync", d["e2e"]["sync_call"]["ms_per_step"], "prep", d["setup_s"])
    print(d["pass_profile"])
except Exception as e:
    print("bench parse failed", e)
PY
tail -3 gpurun_out/bench5.err
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest5.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest5.log; tail -8 gpurun_out/pytest5.log
