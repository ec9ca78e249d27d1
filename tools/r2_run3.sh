mkdir -p gpurun_out
python tools/stress_debug.py 131 > gpurun_out/dbg131.log 2>&1; echo "dbg rc=$?"; cat gpurun_out/dbg131.log
python tools/tune_fit.py run > gpurun_out/tune_planted.log 2>&1; echo "tune rc=$?"; cat gpurun_out/tune_planted.log
L0S_TUNE_Y=random python tools/tune_fit.py run > gpurun_out/tune_random.log 2>&1; echo "tune rc=$?"; cat gpurun_out/tune_random.log
