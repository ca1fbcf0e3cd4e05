#!/bin/bash
# One bench line per workload (BASELINE configs 1-5) under gpurun: gpurun_out/wl/<name>.json
mkdir -p gpurun_out/wl
for w in cfg1 cfg2 cfg3 ladder hanoi elevator deep stair; do
  timeout -k 5 600 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/wl/$w.json 2> gpurun_out/wl/$w.err
done
timeout -k 5 1200 python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/wl/cfg5.json 2> gpurun_out/wl/cfg5.err
ls -la gpurun_out/wl
