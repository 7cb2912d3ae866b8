#!/bin/bash
# compute-sanitizer over the engine (via gpurun): memcheck, synccheck, racecheck, initcheck on a
# C2-shape run with graphs + PDL + the side-stream planner, the planner fork-at-start variant,
# an eager run and a multi-wavelength objective.  Logs in gpurun_out/san/.
E=gpurun_out/san
mkdir -p $E
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
run() {  # tool tag args...
  local tool=$1 tag=$2; shift 2
  timeout 1500 $CS --tool $tool python tools/sanitize.py "$@" > $E/${tool}_${tag}.log 2>&1
  echo "EXIT=$?" >> $E/${tool}_${tag}.log
}
python tools/sanitize.py --gens 30 > $E/plain_default.log 2>&1
python tools/sanitize.py --gens 30 --env QPM_WOLF=planner,QPM_PLAN_FORK=start > $E/plain_planner_start.log 2>&1
for tool in memcheck synccheck racecheck initcheck; do
  run $tool default --gens 30
  run $tool planner_start --gens 30 --env QPM_WOLF=planner,QPM_PLAN_FORK=start
done
run memcheck eager --gens 12 --eager
run memcheck multi --gens 6 --np 256 --d 4000 --nwl 3
run racecheck multi --gens 6 --np 256 --d 4000 --nwl 3
run memcheck de --gens 10 --algo de
run memcheck gwo --gens 10 --algo gwo
echo DONE > $E/done
