timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo PYTEST_RC=$? >> gpurun_out/pytest_gpu.log
python tools/gen_sweep.py "" "QPM_WOLF=planner,QPM_PLAN_FORK=trial,QPM_PLAN_CTAS=444" > gpurun_out/gs.log 2>&1
