# interleaved timing of the tune_fit variants (L0S_TUNE_ROUNDS rounds, min kept), C3 random / planted y, 4 and 2 tasks
for y in random planted; do for t in 4 2; do
  echo "== $y T=$t"; L0S_TUNE_ROUNDS=${ROUNDS:-3} L0S_TUNE_T=$t L0S_TUNE_Y=$y timeout 900 python tools/tune_fit.py run 2>&1 | tail -4 | grep -v agree
done; done
