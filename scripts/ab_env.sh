#!/bin/bash
# A/B a library env knob on the config-3 bench: scripts/ab_env.sh "VAR=a" "VAR=b" [reps]
reps=${3:-2}
for i in $(seq $reps); do
  for e in "$1" "$2"; do
    env $e timeout -k 5 200 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys;d=json.loads(sys.stdin.read());print('$e', round(d['ms_per_step'],2), d['config']['inner_iters'], {k:(round(v['ms_per_launch']*v['launches'],2),v['launches']) for k,v in d['roofline']['phases'].items() if v['launches']})"
  done
done
