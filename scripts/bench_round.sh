#!/bin/bash
# all config bench lines of a round (1 B200): gpurun_out/r02_cfg{1..5}.json
mkdir -p gpurun_out
python bench.py --config 1 --steps 2000 --warmup 20 --secondary 0 > gpurun_out/r02_cfg1.json 2> gpurun_out/r02_cfg1.err
python bench.py --config 2 --steps 20 --warmup 3 > gpurun_out/r02_cfg2.json 2> gpurun_out/r02_cfg2.err
python bench.py --config 3 --steps 3 --warmup 1 --secondary 0 > gpurun_out/r02_cfg3.json 2> gpurun_out/r02_cfg3.err
python bench.py --config 5 --steps 3 --warmup 1 --secondary 0 > gpurun_out/r02_cfg5.json 2> gpurun_out/r02_cfg5.err
python bench.py --config 4 --steps 2 --warmup 1 --secondary 0 --no-cpu-baseline > gpurun_out/r02_cfg4.json 2> gpurun_out/r02_cfg4.err
python bench.py --impl reference --config 2 --steps 3 --warmup 1 > gpurun_out/r02_cfg2_ref.json 2> gpurun_out/r02_cfg2_ref.err
for c in 1 2 3 4 5; do echo "cfg$c: $(head -c 300 gpurun_out/r02_cfg$c.json)"; done
