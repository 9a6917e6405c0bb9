#!/bin/bash
# One GPU session: GPU tests, bench line, ncu launch list, ncu --set full captures
# of the fine CF pass (roofline kernel) and the dominant coarse GMRES passes.
# Outputs in gpurun_out/.  Usage: bash tools/gpu_round.sh [passes...]
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
passes=${@:-L0.CF L0.FC L2.FR L3.FC L1.FR}
for pass in $passes; do
  tag=cfg2_$(echo $pass | tr -d .)
  timeout 600 bash tools/ncu_pass.sh cfg2 $pass $tag
  python tools/ncu_src_summary.py gpurun_out/${tag}_source.csv 25 > gpurun_out/${tag}_source_stalls.txt 2>&1
  python tools/ncu_inst_summary.py gpurun_out/${tag}_source.csv 25 > gpurun_out/${tag}_source_inst.txt 2>&1
done
