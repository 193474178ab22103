#!/bin/bash
# ncu launch list of one whole COCG step (config $1, default 3): per-kernel totals and shares
mkdir -p gpurun_out
c=${1:-3}
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_cg -c ${2:-12000} --csv \
    --log-file gpurun_out/launches_cfg${c}.csv python scripts/cfg_step.py $c > gpurun_out/ncu_launch_cfg${c}.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_cfg${c}.csv > gpurun_out/launches_cfg${c}_summary.txt 2>&1
cat gpurun_out/launches_cfg${c}_summary.txt
