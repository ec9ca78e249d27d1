mkdir -p gpurun_out
timeout 900 python tools/tune_fit.py run > gpurun_out/tune17_planted.txt 2>&1; echo "planted rc=$?"; cat gpurun_out/tune17_planted.txt
L0S_TUNE_Y=random timeout 900 python tools/tune_fit.py run > gpurun_out/tune17_random.txt 2>&1; echo "random rc=$?"; cat gpurun_out/tune17_random.txt
