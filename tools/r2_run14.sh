mkdir -p gpurun_out
for T in 1 2 8; do
L0S_TUNE_T=$T timeout 900 python tools/tune_fit.py run > gpurun_out/tune14_T$T.txt 2>&1; echo "T=$T rc=$?"; cat gpurun_out/tune14_T$T.txt
done
