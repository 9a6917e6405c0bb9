#!/bin/bash
# One GPU session: bench line, ncu launch list, ncu --set full captures of the
# fine CF pass and the coarse GMRES passes.  Outputs in gpurun_out/.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
for pass in L0.CF L0.FC L3.FC L2.FC L1.FC; do
  tag=cfg2_$(echo $pass | tr -d .)
  timeout 600 bash tools/ncu_pass.sh cfg2 $pass $tag
  python tools/ncu_src_summary.py gpurun_out/${tag}_source.csv 25 > gpurun_out/${tag}_source_stalls.txt 2>&1
  python tools/ncu_inst_summary.py gpurun_out/${tag}_source.csv 25 > gpurun_out/${tag}_source_inst.txt 2>&1
done
