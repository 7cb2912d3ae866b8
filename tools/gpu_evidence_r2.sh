#!/bin/bash
# Round-2 evidence in one GPU call (outputs in gpurun_out/ev2/): parity suite, bench at the
# driver's settings and a long run, reference arm, BASELINE configs, e2e probe, launch list of
# the bench command, ncu --set full of a late C2 generation, a C3 generation, C4 run_gwo,
# C5 fitness, and the multi-GPU shard probe (emulated ranks + NCCL-rate exchange model).
E=gpurun_out/${EV:-ev3}
mkdir -p $E
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $E/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > $E/pytest_gpu.log 2>&1; echo RC=$? >> $E/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > $E/bench_20_5.jsonl 2> $E/bench_20_5.err
timeout 900 python bench.py --steps 950 --warmup 50 --no-cpu-baseline > $E/bench_950_50.jsonl 2> $E/bench_950.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $E/bench_reference.jsonl 2>&1
for a in "c1 hybrid" "c2 hybrid" "c3 hybrid" "c4 hybrid" "c4 de" "c4 gwo" "c5 hybrid"; do
  set -- $a
  timeout 300 python tools/run_config.py --config $1 --algo $2 --gens 20 --warm 20 --profile 0 >> $E/configs.jsonl 2>> $E/configs.err
done
timeout 300 python tools/e2e_probe.py --gens 20 --reps 3 > $E/e2e_probe.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches_bench.csv \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $E/ncu_launch.log 2>&1
KRE="k_de_trial|k_gwo_apply|k_fit_fast|k_finish_select"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRE}" -s 3600 -c 6 \
  -o $E/prof_c2_gen python tools/prof_engine.py --gens 1 --warm 600 > $E/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_de_trial|k_fit_fast|k_gwo_apply|k_select|k_fit_finish" -s 43 -c 8 \
  -o $E/prof_c3_gen python tools/prof_engine.py --gens 1 --warm 5 --np 8192 --d 100000 > $E/ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gwo_continuous|k_fit_fast|k_select_stats|k_topk" -s 42 -c 4 \
  -o $E/prof_c4_gwo python tools/prof_engine.py --gens 1 --warm 10 --np 4096 --d 10000 --algo gwo > $E/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fit_fast -s 2 -c 1 \
  -o $E/prof_fit_c5 python tools/bench_fitness.py --rows 4092 --d 20000 --nwl 64 --iters 3 > $E/ncu_fit.log 2>&1
for w in 2 4 8; do timeout 400 python tools/shard_probe.py --world $w --seg-chunks 2 >> $E/shard_probe.jsonl 2>> $E/shard_probe.err; done
timeout 900 python tools/shard_probe.py --world 8 --np 8192 --d 100000 --t 0.1 --warm 5 --gens 5 >> $E/shard_probe.jsonl 2>> $E/shard_probe.err
[ -f build/ab/libqpm_trace.so ] && timeout 300 python tools/timeline.py > $E/timeline.log 2>&1
timeout 300 python tools/timeline.py build/ab/libqpm_trace.so --warm 5 --gens 20 > $E/timeline_early.log 2>&1
echo DONE > $E/done
