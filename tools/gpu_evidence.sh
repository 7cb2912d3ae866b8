#!/bin/bash
# The round's evidence in one GPU call: parity tests, bench (+ reference arm),
# BASELINE configs, §8(f) extras, device timeline, ncu launch list, ncu --set full
# of a late C2 generation and of the C5-shape fitness kernel.  Outputs in gpurun_out/ev/.
# usage (via gpurun): bash tools/gpu_evidence.sh   (build/ab/libqpm_trace.so must exist for the timeline)
E=gpurun_out/ev
mkdir -p $E
timeout 1200 python -m pytest tests -m gpu -q > $E/pytest_gpu.log 2>&1; echo RC=$? >> $E/pytest_gpu.log
timeout 600 python bench.py > $E/bench.jsonl 2> $E/bench.err; echo RC=$? >> $E/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $E/bench_reference.jsonl 2>&1
for a in "c1 hybrid" "c2 hybrid" "c3 hybrid" "c4 hybrid" "c4 de" "c4 gwo" "c5 hybrid"; do
  set -- $a
  timeout 300 python tools/run_config.py --config $1 --algo $2 --gens 20 --warm 20 --profile 0 >> $E/configs.jsonl 2>> $E/configs.err
done
timeout 300 python tools/measure_extras.py > $E/extras.log 2>&1
[ -f build/ab/libqpm_trace.so ] && timeout 300 python tools/timeline.py > $E/timeline.log 2>&1
python tools/prof_engine.py --gens 2 > $E/prof_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches.csv \
    python tools/prof_engine.py --gens 2 > $E/ncu_launch.log 2>&1
# C2 (NP 1024): k_de_trial, k_fit_fast x2, k_finish_select x2, k_gwo_apply per generation
KRE="k_de_trial|k_gwo_apply|k_fit_fast|k_finish_select|k_fit_finish|k_select_stats|k_select_topk"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRE}" -s 3600 -c 6 \
  -o $E/prof_gen python tools/prof_engine.py --gens 1 --warm 600 > $E/ncu_gen.log 2>&1
python tools/bench_fitness.py --rows 4092 --d 20000 --nwl 64 --iters 3 > $E/fit_c5_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fit_fast -s 2 -c 1 \
    -o $E/prof_fit_c5 python tools/bench_fitness.py --rows 4092 --d 20000 --nwl 64 --iters 3 > $E/ncu_fit.log 2>&1
# the bench's multi-GPU runs use 2-chunk fitness segments (even C2 split)
for w in 2 4 8; do timeout 400 python tools/shard_probe.py --world $w --seg-chunks 2 >> $E/shard_probe.jsonl 2>> $E/shard_probe.err; done
timeout 900 python tools/shard_probe.py --world 8 --d 100000 --warm 5 --gens 5 >> $E/shard_probe.jsonl 2>> $E/shard_probe.err
echo DONE >> $E/pytest_gpu.log
