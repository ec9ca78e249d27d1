mkdir -p gpurun_out
python tools/stress_debug.py 131 > gpurun_out/dbg131.log 2>&1; echo "dbg rc=$?"; grep -v "^[0-9]" gpurun_out/dbg131.log
python tools/tune_fit.py run > gpurun_out/tune_planted.log 2>&1; echo "tune rc=$?"; cat gpurun_out/tune_planted.log
L0S_TUNE_Y=random python tools/tune_fit.py run > gpurun_out/tune_random.log 2>&1; echo "tune rc=$?"; cat gpurun_out/tune_random.log
bash tools/ncu_fit.sh r2b_fit3_planted > /dev/null 2>&1; echo ncu1 $?
ncu -i gpurun_out/r2b_fit3_planted.ncu-rep --page source --csv --print-source sass > gpurun_out/r2b_fit3_planted_src.csv 2>/dev/null
cat gpurun_out/r2b_fit3_planted_summary.txt
