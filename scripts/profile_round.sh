#!/bin/bash
# Profiling pass for profiles/<round>/ (run under gpurun on one B200).
#  1. bench line (CUDA events, not under a profiler)
#  2. ncu launch list of one config-3 solve (host-driven loop: ncu cannot profile kernel
#     nodes of graphs with conditional nodes; the same kernels; cold-cache,
#     serialised launches: compare shares, not absolute times)
#  3. ncu --set full of one mid-solve launch of each top kernel
#  4. the Bellman-Ford arm: launch list of its rounds + one full capture
#  5. PGSI_TRACE=2 phase times inside k_inc_iter over one solve
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
timeout -k 5 600 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum
PGSI_DEVICE_LOOP=0 timeout -k 5 900 ncu --metrics $M --clock-control none -c 3000 --csv --log-file $OUT/launches.csv \
    python bench.py --profile --steps 1 --warmup 0 > $OUT/launches.log 2>&1
for k in k_inc_iter k_v2_cpx k_switch k_v1; do
  PGSI_DEVICE_LOOP=0 timeout -k 5 900 ncu --set full --clock-control none --import-source on -k regex:"^${k}\$" -s 8 -c 1 \
      -o $OUT/full_$k python bench.py --profile --steps 1 --warmup 0 > $OUT/full_$k.log 2>&1
done
timeout -k 5 600 ncu --metrics $M --clock-control none -k regex:k_bf_round -s 100 -c 200 --csv \
    --log-file $OUT/launches_bf.csv python scripts/arms_probe.py 10000000 32 bf > $OUT/launches_bf.log 2>&1
timeout -k 5 600 ncu --set full --clock-control none --import-source on -k regex:k_bf_round -s 400 -c 1 \
    -o $OUT/full_k_bf_round python scripts/arms_probe.py 10000000 32 bf > $OUT/full_k_bf_round.log 2>&1
PGSI_TRACE=2 timeout -k 5 300 python scripts/trace_solve.py > /dev/null 2> $OUT/inc_phase_trace.txt
ls -la $OUT
