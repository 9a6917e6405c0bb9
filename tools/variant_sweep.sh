#!/bin/bash
# Per-pass timings of cfg2 under launch-variant overrides (env), one bench run each.
# Usage: bash tools/variant_sweep.sh "ENV1=.. ENV2=.." "ENV=.." ...   (outputs in gpurun_out/sweep_*.json)
i=0
for envs in "$@"; do
  i=$((i+1))
  env $envs timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sweep_$i.json 2> gpurun_out/sweep_$i.err
  python - "$envs" gpurun_out/sweep_$i.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
p = d["passes"]
lv = {}
for k, v in p.items():
    lv.setdefault(k.split(".")[0], 0.0)
    lv[k.split(".")[0]] += v["ms"]
print(f"[{sys.argv[1]}] ms/solve {d['ms_per_step']:.2f} iters {d['config']['iterations']} ratio {d['config']['final_ratio']:.3e} | " +
      " ".join(f"{k}={v/11:.3f}" for k, v in sorted(lv.items())) + " | " +
      " ".join(f"{k}={v['ms']/v['launches']:.3f}" for k, v in sorted(p.items()) if k[:2] in ("L1", "L2", "L3")))
PY
done
