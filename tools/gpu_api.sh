# pipelined e2e: quick 1-rank bench (C5 + parity) and the 2-rank functional run on one GPU
timeout 1200 python bench.py --steps 3 --warmup 3 --legs none --no-cpu-baseline > gpurun_out/e2e1.json 2> gpurun_out/e2e1.err; echo rc=$?
timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 --legs none --no-cpu-baseline > gpurun_out/e2e2.json 2> gpurun_out/e2e2.err; echo rc=$?
python - <<'PY'
import json
for f in ("gpurun_out/e2e1.json", "gpurun_out/e2e2.json"):
    d = json.load(open(f))
    print(f, d["n_gpus"], round(d["value"] / 1e9, 3), round(d["e2e"]["value"] / 1e9, 3), d["e2e"]["ms_per_step"], d["ms_per_step"], d["parity"]["match"])
PY
