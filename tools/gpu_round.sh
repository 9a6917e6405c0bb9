#!/bin/bash
# One GPU session: tests, bench, launch list, ncu captures.  Outputs in gpurun_out/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_target.py cfg2 L0.CF > gpurun_out/t1.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 -o gpurun_out/cfg2_L0CF -f \
    python tools/ncu_target.py cfg2 L0.CF > gpurun_out/ncu_full1.log 2>&1; echo "ncu full1 rc=$?"
python tools/ncu_target.py cfg2 L3.FC > gpurun_out/t2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 -o gpurun_out/cfg2_L3FC -f \
    python tools/ncu_target.py cfg2 L3.FC > gpurun_out/ncu_full2.log 2>&1; echo "ncu full2 rc=$?"
