#!/bin/bash
# ncu evidence for profiles/ (one GPU): launch list of cfg2 steps, thread-level FP64
# instruction counts and full captures (with SASS-level source pages) of the level-0
# kernels (cfg2), full captures of the width-64 COCG kernels (cfg3 windowed spmv and TMA
# update, cfg5 windowed spmv, and the staged gather spmv as the A/B partner).
set -u
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --secondary 0 \
    > gpurun_out/ncu_launch_cfg2.log 2>&1; echo "launch list rc=$?"
ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
    --clock-control none -k regex:k_l0_ -c 3 --csv --log-file gpurun_out/l0_fp64_counts.csv \
    python scripts/cfg_step.py 2 > gpurun_out/ncu_fp64.log 2>&1; echo "fp64 counts rc=$?"
for k in k_l0_k2 k_l0_k3 k_l0_s1; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 0 -c 1 \
      -o gpurun_out/cfg2_$k -f python scripts/cfg_step.py 2 > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
  ncu -i gpurun_out/cfg2_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/cfg2_${k}_sass.csv 2>/dev/null
done
for k in k_cg_spmv_win k_cg_update_tma; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 \
      -o gpurun_out/cfg3_$k -f python scripts/cfg_step.py 3 > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:k_cg_spmv_win -s 4 -c 1 \
    -o gpurun_out/cfg5_k_cg_spmv_win -f python scripts/cfg_step.py 5 > gpurun_out/ncu_cfg5_spmv.log 2>&1; echo "cfg5 spmv rc=$?"
REXI_COCG_NOTMA=1 ncu --set full --clock-control none --import-source on -k regex:k_cg_spmv_st -s 4 -c 1 \
    -o gpurun_out/cfg3_k_cg_spmv_st -f python scripts/cfg_step.py 3 > gpurun_out/ncu_spmv_st.log 2>&1; echo "cfg3 spmv_st rc=$?"
for r in gpurun_out/*.ncu-rep; do python scripts/ncu_summary.py raw $r; done > gpurun_out/ncu_raw_summaries.txt 2>&1
for r in gpurun_out/cfg3_k_cg_spmv_win.ncu-rep gpurun_out/cfg3_k_cg_update_tma.ncu-rep gpurun_out/cfg5_k_cg_spmv_win.ncu-rep; do
  ncu -i $r --page details --csv > ${r%.ncu-rep}_details.csv 2>/dev/null
done
