#!/bin/bash
# One GPU session: GPU tests, bench lines (cfg4 headline, cfg2/cfg3 secondary), ncu
# launch list, ncu --set full captures of the named passes of one config.
# Outputs in gpurun_out/.  Usage: bash tools/gpu_round.sh [cfg [passes...]]
cfg=${1:-cfg4}; shift
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_cfg4.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
for c in cfg2 cfg3 cfg1; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2>> gpurun_out/bench.err; echo "bench $c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2>> gpurun_out/bench.err; echo "ref rc=$?"
timeout 300 python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$cfg.csv \
    python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
python tools/launch_summary.py gpurun_out/launches_$cfg.csv > gpurun_out/launch_summary_$cfg.txt
passes=${@:-L0.CF L0.FC L1.FR L2.FR L3.FC}
for pass in $passes; do
  tag=${cfg}_$(echo $pass | tr -d .)
  timeout 900 bash tools/ncu_pass.sh $cfg $pass $tag
  python tools/ncu_src_summary.py gpurun_out/${tag}_source.csv 25 > gpurun_out/${tag}_source_stalls.txt 2>&1
  python tools/ncu_inst_summary.py gpurun_out/${tag}_source.csv 25 > gpurun_out/${tag}_source_inst.txt 2>&1
  rm -f gpurun_out/${tag}_source.csv
done
# extra captures of the other configs' fine passes + the parity report
for cp in cfg2:L0.CF cfg3:L0.FC; do
  c=${cp%%:*}; pass=${cp##*:}; tag=${c}_$(echo $pass | tr -d .)
  timeout 900 bash tools/ncu_pass.sh $c $pass $tag
  python tools/ncu_src_summary.py gpurun_out/${tag}_source.csv 25 > gpurun_out/${tag}_source_stalls.txt 2>&1
  python tools/ncu_inst_summary.py gpurun_out/${tag}_source.csv 25 > gpurun_out/${tag}_source_inst.txt 2>&1
  rm -f gpurun_out/${tag}_source.csv
done
timeout 1500 python tools/parity_report.py > gpurun_out/parity.json 2> gpurun_out/parity.err; echo "parity rc=$?"
