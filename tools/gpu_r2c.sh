mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-paths > gpurun_out/bench3.json 2> gpurun_out/bench3.err
echo "bench rc=$?" >> gpurun_out/bench3.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench3.json").read())
print("ids ms", d["ms_per_step"], "count ms", d["modes"]["count"]["ms_per_step"], "e2e", d["e2e"]["ms_per_step"],
      "sync", d["e2e"]["sync_call"]["ms_per_step"], "prep", d["setup_s"])
print(d["pass_profile"])
PY
