#!/bin/bash
# Alternating A/B of library builds (drift-robust): REPS rounds of every
# build/ab/libqpm_*.so and the in-tree library, one C2 gen_sweep each.
# usage (via gpurun): REPS=4 bash tools/ab_alt.sh [gen_sweep config]
REPS=${REPS:-4}
for r in $(seq $REPS); do
  for lib in paper_2511_01255_b200/libqpm_b200.so build/ab/libqpm_*.so; do
    printf "%-40s " "$(basename $lib)"
    QPM_LIB=$lib timeout 300 python tools/gen_sweep.py "$@" 2>&1 | tail -1 | awk '{print $2, $3}'
  done
done
