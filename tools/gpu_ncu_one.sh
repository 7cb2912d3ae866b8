#!/bin/bash
# --set full capture of one kernel of a late C2 generation.
# usage (via gpurun): bash tools/gpu_ncu_one.sh TAG KERNEL_REGEX [WARM] [COUNT]
TAG=$1; KRE=$2; WARM=${3:-600}; CNT=${4:-1}
mkdir -p gpurun_out
python tools/prof_engine.py --gens 1 --warm $WARM > gpurun_out/prof_plain_${TAG}.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRE}" -s $((WARM * ${PER:-1})) -c $CNT \
    -o gpurun_out/prof_${TAG} python tools/prof_engine.py --gens 1 --warm $WARM > gpurun_out/ncu_${TAG}.log 2>&1
echo NCU_RC=$? >> gpurun_out/ncu_${TAG}.log
