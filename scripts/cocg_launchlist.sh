#!/bin/bash
# ncu launch list of a window of a COCG step's launches (narrow phase): config, skip, count
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_cg -s ${2:-10000} -c ${3:-600} --csv \
    --log-file gpurun_out/launches_cfg$1_narrow.csv python scripts/cfg_step.py $1 > gpurun_out/ncu_launch_cfg$1.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_cfg$1_narrow.csv
