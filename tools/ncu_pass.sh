#!/bin/bash
# ncu --set full of one relax pass: tools/ncu_pass.sh cfg2 L0.FC tag
cfg=$1; pass=$2; tag=$3
python tools/ncu_target.py $cfg $pass > gpurun_out/${tag}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 -o gpurun_out/${tag} -f \
    python tools/ncu_target.py $cfg $pass > gpurun_out/${tag}_ncu.log 2>&1; echo "ncu $tag rc=$?"
ncu -i gpurun_out/${tag}.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv 2>/dev/null
ncu -i gpurun_out/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_source.csv 2>/dev/null
# keep the call's output under gpurun's 64 MiB merge limit: the CSV pages above are what is read
rm -f gpurun_out/${tag}.ncu-rep gpurun_out/${tag}_details.csv
