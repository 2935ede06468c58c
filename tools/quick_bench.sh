#!/bin/bash
# quick per-kernel timing of the bench workload (no sweep / CPU baseline)
timeout 300 python bench.py --sweep-steps 0 --no-cpu-baseline "$@" > gpurun_out/qb.json 2>gpurun_out/qb.err || tail -5 gpurun_out/qb.err
python - <<'PY'
import json; d=json.load(open("gpurun_out/qb.json"))
print("value", round(d["value"]), "e2e", round(d["e2e"]["value"]) if d.get("e2e") else None, "dense", round(d["dense_path_fps"] or 0))
for k in d["roofline"]["top_kernels"]: print(f'{k["kernel"]:12s} {k["ms_per_launch"]*1000:8.1f} us  frac {k["roofline_frac"]:.3f}')
print("ms/step", round(d["ms_per_step"], 4), {k: v["us"] for k, v in d["roofline"]["all_kernels"].items()})
PY
