# run the tune_fit variants on C3 planted and random y, 4 / 2 / 1 tasks (gpurun)
mkdir -p gpurun_out
for y in planted random; do for t in 4 2 1; do
  echo "== $y T=$t"; L0S_TUNE_T=$t L0S_TUNE_Y=$y timeout 900 python tools/tune_fit.py run 2>&1 | tail -3
done; done
