timeout 900 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_gpu.log 2>&1; echo PYTEST_RC=$? >> gpurun_out/pytest_gpu.log
python tools/gen_sweep.py "QPM_WOLF=fused" "" > gpurun_out/gs.log 2>&1
QPM_NVCC_EXTRA=-DQPM_DE_MINB=4 python -m paper_2511_01255_b200.build --force > /dev/null 2>&1
echo minb4 >> gpurun_out/gs.log; python tools/gen_sweep.py "QPM_WOLF=fused" "" >> gpurun_out/gs.log 2>&1
