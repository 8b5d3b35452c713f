mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 1 --steps 3 --warmup 3 --force-merge --no-cpu-baseline --no-paths > gpurun_out/tr2.log 2> gpurun_out/tr2.err
echo "torchrun rc=$?" >> gpurun_out/tr2.err; tail -n 2 gpurun_out/tr2.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/tr2.log").read().strip().splitlines()[-1])
print("host_gather", d["host_gather"]); print("id_exchange", d["id_exchange"]["ms_per_step"]); print("e2e", d["e2e"]["ms_per_step"])
PY
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "sharded or sorted or c3" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt.log; tail -n 3 gpurun_out/pt.log
timeout 900 python tools/bench_configs.py c3 > gpurun_out/c3.json 2> gpurun_out/c3.err; python - <<'PY'
import json
d = json.load(open("gpurun_out/c3.json"))[0]
print({p: {k: v for k, v in e.items() if "us_per" in k} for p, e in d["paths"].items()})
PY
