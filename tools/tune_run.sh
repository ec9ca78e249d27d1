# run the tune_fit variants on C3 planted and random y (gpurun)
mkdir -p gpurun_out
for y in planted random; do echo "== $y"; L0S_TUNE_Y=$y timeout 900 python tools/tune_fit.py run 2>&1 | tail -8; done
