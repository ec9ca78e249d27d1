# interleaved timing of the tune_fit variants on C3 planted y, 4 and 2 tasks
for t in 4 2; do
  echo "== planted T=$t"; L0S_TUNE_ROUNDS=${ROUNDS:-2} L0S_TUNE_T=$t L0S_TUNE_Y=planted timeout 900 python tools/tune_fit.py run 2>&1 | tail -7 | grep -v agree
done
