mkdir -p gpurun_out
python tools/tune_fit.py run > gpurun_out/tune_planted.log 2>&1; echo "tune rc=$?"; cat gpurun_out/tune_planted.log
L0S_TUNE_Y=random python tools/tune_fit.py run > gpurun_out/tune_random.log 2>&1; echo "tune rc=$?"; cat gpurun_out/tune_random.log
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.txt 2>&1; echo "e2e rc=$?"; cat gpurun_out/e2e_probe.txt
