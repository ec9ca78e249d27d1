mkdir -p gpurun_out
timeout 900 python tools/tune_fit.py run > gpurun_out/tune16_planted.txt 2>&1; echo "planted rc=$?"; cat gpurun_out/tune16_planted.txt
L0S_TUNE_Y=random timeout 900 python tools/tune_fit.py run > gpurun_out/tune16_random.txt 2>&1; echo "random rc=$?"; cat gpurun_out/tune16_random.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/r2c_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r2c_tests.log
