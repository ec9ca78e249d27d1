mkdir -p gpurun_out
python tools/dbg/stress131.py 131 > gpurun_out/dbg131.log 2>&1; echo "dbg rc=$?"; cat gpurun_out/dbg131.log
bash tools/ncu_fit.sh r2a_fit3_planted > /dev/null 2>&1; echo ncu1 $?
L0S_TUNE_Y=random bash tools/ncu_fit.sh r2a_fit3_random > /dev/null 2>&1; echo ncu2 $?
for t in r2a_fit3_planted r2a_fit3_random; do ncu -i gpurun_out/$t.ncu-rep --page source --csv --print-source sass > gpurun_out/${t}_src.csv 2>/dev/null; done
cat gpurun_out/r2a_fit3_planted_summary.txt gpurun_out/r2a_fit3_random_summary.txt
ls -la gpurun_out
