#!/bin/bash
# Sweep the side-stream planner placement (QPM_PLAN_FORK) and CTA count (QPM_PLAN_CTAS) on the C2 bench.
# usage (via gpurun): bash tools/plan_sweep.sh "start trial" "148 296 592 1184"
FORKS=${1:-"start trial"}
CTAS=${2:-"148 296 592 1184"}
mkdir -p gpurun_out
for f in $FORKS; do
  for n in $CTAS; do
    r=$(QPM_PLAN_FORK=$f QPM_PLAN_CTAS=$n timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), 'us/gen', [(s['name'], round(s['ms']*1000,1)) for s in d['stages']])")
    echo "fork=$f ctas=$n $r"
  done
done
