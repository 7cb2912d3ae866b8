#!/bin/bash
# final round-2 evidence (outputs in gpurun_out/fin/)
E=gpurun_out/${EV:-fin}
mkdir -p $E
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $E/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > $E/pytest_gpu.log 2>&1; echo RC=$? >> $E/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $E/smoke.log 2>&1; echo RC=$? >> $E/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $E/bench_20_5.jsonl 2> $E/bench_20_5.err
timeout 900 python bench.py --steps 950 --warmup 50 --no-cpu-baseline > $E/bench_950_50.jsonl 2> $E/bench_950.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $E/bench_reference.jsonl 2> $E/bench_reference.err
timeout 300 python tools/spectrum_probe.py > $E/spectrum_probe.jsonl 2>&1
timeout 300 python tools/e2e_detail.py > $E/e2e_detail.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches_bench.csv \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $E/ncu_launch.log 2>&1
echo DONE > $E/done
