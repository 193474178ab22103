#!/bin/bash
# COCG: windowed spmv down to kp = 16 / 32 (REXI_COCG_WINMIN) and the TMA update
# (REXI_COCG_NOUTMA=1: off); bitwise comparison, cfg 3 step times, per-width profile
mkdir -p gpurun_out
run() {
  timeout 300 python scripts/cocg_snapshot.py gpurun_out/snap_$1.npz 2>&1 | tail -1
  timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
}
python paper_1912_03312_b200/build_native.py > /dev/null 2>&1
echo "=== win >= 64, update old"; REXI_COCG_WINMIN=64 REXI_COCG_NOUTMA=1 run base
echo "=== win >= 64, update TMA"; REXI_COCG_WINMIN=64 run utma
echo "=== win >= 32, update TMA"; REXI_COCG_WINMIN=32 run w32
echo "=== win >= 16, update TMA"; run w16
for v in utma w32 w16; do python scripts/cocg_compare.py gpurun_out/snap_base.npz gpurun_out/snap_$v.npz; done
REXI_COCG_TRACE=1 timeout 300 python scripts/cocg_widths.py 3 2 2>&1 | grep "cg_"
echo "=== cfg4"; timeout 600 python scripts/cocg_steps.py 4 2 2>&1 | grep "^step"
echo "=== cfg5"; timeout 600 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step"
timeout 900 python -m pytest tests/test_gpu_cocg_layout.py tests/test_gpu_stiff.py tests/test_gpu_hygiene.py tests/test_gpu_distributed.py -x -q 2>&1 | tail -3
