#!/bin/bash
# One GPU round trip: parity tests, bench, launch list, full ncu of the hot kernels.
# usage (via gpurun): bash tools/gpu_cycle.sh [tag] [ncu-kernel-regex] [launches|full]
# Only one ncu pass per call: "launches" (default) = the launch list, "full" = --set full capture.
TAG=${1:-cycle}
KRE=${2:-"k_de_trial|k_gwo_apply|k_fit_fast|k_fit_finish|k_select_stats|k_select_topk"}
NCU=${3:-launches}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo PYTEST_RC=$? >> gpurun_out/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/bench.log 2>&1; echo BENCH_RC=$? >> gpurun_out/bench.log
if [ "$NCU" = launches ]; then
python tools/prof_engine.py --gens 2 > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python tools/prof_engine.py --gens 2 > gpurun_out/ncu_launch.log 2>&1
echo NCU1_RC=$? >> gpurun_out/ncu_launch.log
else
python tools/prof_engine.py --gens 1 --warm 0 > gpurun_out/prof_plain1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRE}" -s 2 -c 8 -o gpurun_out/prof_${TAG} python tools/prof_engine.py --gens 1 --warm 0 > gpurun_out/ncu_full.log 2>&1
echo NCU2_RC=$? >> gpurun_out/ncu_full.log
fi
