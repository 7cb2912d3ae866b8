#!/bin/bash
# One --set full ncu capture of a C2 generation (late phase: 600 graph-replayed
# warm-up generations, then one eager generation whose 8 main-chain kernels are
# captured).  usage (via gpurun): bash tools/gpu_ncu_full.sh TAG [WARM]
TAG=${1:-full}
WARM=${2:-600}
KRE="k_de_trial|k_gwo_apply|k_fit_fast|k_fit_finish|k_select_stats|k_select_topk"
mkdir -p gpurun_out
python tools/prof_engine.py --gens 1 --warm $WARM > gpurun_out/prof_plain_full.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRE}" -s $((WARM * 8)) -c 8 \
    -o gpurun_out/prof_${TAG} python tools/prof_engine.py --gens 1 --warm $WARM > gpurun_out/ncu_full_${TAG}.log 2>&1
echo NCU_RC=$? >> gpurun_out/ncu_full_${TAG}.log
