#!/bin/bash
# A/B builds of libpgsi.so on a bench workload (run under gpurun):
#   REPS=2 ARGS="--workload cfg3" scripts/ab_lib.sh A.so B.so [C.so ...]
# Each variant is copied over paper_1705_02313_b200/libpgsi.so before its runs.
reps=${REPS:-2}
L=paper_1705_02313_b200/libpgsi.so
cp $L /tmp/ab_orig.so
for i in $(seq $reps); do
  for v in "$@"; do
    cp $v $L
    timeout -k 5 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-arms $ARGS 2>/dev/null | tail -1 | \
      python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v'.split('/')[-1], round(d['ms_per_step'],3), d['config'].get('inner_iters'), {k:(round(v['ms_per_launch']*v['launches'],2),v['launches']) for k,v in d['roofline']['phases'].items() if v['launches']})"
  done
done
cp /tmp/ab_orig.so $L
