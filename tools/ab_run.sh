#!/bin/bash
# Time every build/ab/libqpm_*.so (plus the in-tree library) on C2 generations.
# usage (via gpurun): bash tools/ab_run.sh [gen_sweep configs...]
mkdir -p gpurun_out
for lib in paper_2511_01255_b200/libqpm_b200.so build/ab/libqpm_*.so; do
  echo "== $lib"
  QPM_LIB=$lib timeout 300 python tools/gen_sweep.py "$@" 2>&1 | tail -5
done
