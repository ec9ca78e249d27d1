mkdir -p gpurun_out
python tools/tune_fit.py run > gpurun_out/tune_planted.log 2>&1; echo "tune rc=$?"; cat gpurun_out/tune_planted.log
L0S_TUNE_Y=random python tools/tune_fit.py run > gpurun_out/tune_random.log 2>&1; echo "tune rc=$?"; cat gpurun_out/tune_random.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/gpu_tests.log
