#!/bin/bash
# Per-pass timings of a config (CFG, default cfg4) under launch-variant overrides (env),
# one bench run each.
# Usage: CFG=cfg4 bash tools/variant_sweep.sh "ENV1=.. ENV2=.." "ENV=.." ...   (outputs in gpurun_out/sweep_*.json)
CFG=${CFG:-cfg4}
i=0
for envs in "$@"; do
  i=$((i+1))
  env $envs timeout 600 python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sweep_$i.json 2> gpurun_out/sweep_$i.err
  python - "$envs" gpurun_out/sweep_$i.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
except Exception as e:
    print(f"[{sys.argv[1]}] FAILED {e}"); sys.exit(0)
p = d["passes"]
it = d["solve"]["iterations"]
lv = {}
for k, v in p.items():
    lv.setdefault(k.split(".")[0], 0.0)
    lv[k.split(".")[0]] += v["ms"]
print(f"[{sys.argv[1]}] ms/solve {d['ms_per_step']:.2f} iters {it} ratio {d['solve']['final_ratio']:.3e} | " +
      " ".join(f"{k}={v:.2f}" for k, v in sorted(lv.items())) + " | " +
      " ".join(f"{k}={v['ms']/v['launches']:.3f}" for k, v in sorted(p.items()) if k[:2] in ("L0", "L1", "L2", "L3")))
PY
done
