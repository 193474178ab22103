#!/bin/bash
# ncu evidence for profiles/ (one GPU): launch list of cfg2 steps, full captures of
# the level-0 kernels (cfg2) and of the width-64 COCG kernels (cfg3).
set -u
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/ncu_launch_cfg2.log 2>&1; echo "launch list rc=$?"
for k in k_l0_k2 k_l0_k3 k_l0_s1; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 0 -c 1 \
      -o gpurun_out/cfg2_$k -f python scripts/cfg_step.py 2 > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
done
for k in k_cg_spmv_st k_cg_update; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 \
      -o gpurun_out/cfg3_$k -f python scripts/cfg_step.py 3 > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
done
