#!/bin/bash
# Config-3 bench under several library env settings (tuning knobs; results never change):
#   scripts/sweep_env.sh "A=1 B=2" "A=3" ...
for e in "$@"; do
  env $e timeout -k 5 200 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys;d=json.loads(sys.stdin.read());print('$e', round(d['ms_per_step'],2), d['config']['inner_iters'], d['config']['incremental_valuations_per_solve'], {k:(round(v['ms_per_launch']*v['launches'],2),v['launches']) for k,v in d['roofline']['phases'].items() if v['launches']})"
done
