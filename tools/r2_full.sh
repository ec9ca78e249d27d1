# Round-2 full measurement pass (run under gpurun; one GPU, never multi-rank).
#   COMMIT=<sha> bash tools/r2_full.sh <tag>
# smoke + GPU tests, ncu captures of HEAD (fit3 planted/random, staging, INT8 Gram) written to
# profiles/fit3_profile.json before the bench reads it, launch list, bench line with clocks,
# reference arm.
set -u
tag=${1:-r2}
commit=${COMMIT:-unknown}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 300 python __graft_entry__.py > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${tag}_smoke.log
  timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider --durations=10 > gpurun_out/${tag}_tests.log 2>&1
  echo "tests rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/${tag}_tests.log | tail -8
fi
# planted y: the tile-screened sweep k_fit3<4, true>; random y: the plain sweep k_fit3<4, false> (the screened
# kernel's CTAs exit at once there -- fit3.cu, k_fit3)
for y in planted random; do
  if [ $y = planted ]; then kre='regex:k_fit3.*bool.1'; kname='k_fit3<4, true> (tile screen)'; else kre='regex:k_fit3.*bool.0'; kname='k_fit3<4, false>'; fi
  L0S_TUNE_Y=$y timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$kre" -s 1 -c 1 -f \
      -o gpurun_out/${tag}_fit3_${y} python tools/tune_fit.py one > gpurun_out/${tag}_fit3_${y}.log 2>&1
  echo "fit3 $y rc=$?"
  python tools/ncu_summary.py gpurun_out/${tag}_fit3_${y}.ncu-rep "${tag} (${commit}): ${kname} on C3, ${y} y" > gpurun_out/${tag}_fit3_${y}_ncu.txt
  ncu -i gpurun_out/${tag}_fit3_${y}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_fit3_${y}_src.csv 2>/dev/null
  python tools/ncu_blocks.py gpurun_out/${tag}_fit3_${y}_src.csv 12 > gpurun_out/${tag}_fit3_${y}_blocks.txt 2>&1
  grep -E "duration|FP64 pipe|occupancy|issue active" gpurun_out/${tag}_fit3_${y}_ncu.txt
done
python tools/ncu_summary.py gpurun_out/${tag}_fit3_planted.ncu-rep x --json "$commit" > gpurun_out/${tag}_fit3_profile.json
cp gpurun_out/${tag}_fit3_profile.json profiles/fit3_profile.json
for k in k_stage_rows k_oz_gemm k_exact_smem; do
  # the third k_stage_rows launch is a feature-row pass (the first of each stage is the property row)
  skip=2; [ $k = k_stage_rows ] && skip=3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -f \
      -o gpurun_out/${tag}_$k python tools/time_stage.py > gpurun_out/${tag}_$k.log 2>&1
  echo "$k full rc=$?"
  python tools/ncu_summary.py gpurun_out/${tag}_$k.ncu-rep "${tag} (${commit}): $k on C3" > gpurun_out/${tag}_${k}_ncu.txt
  grep -E "kernel|duration|DRAM throughput|tensor \(tc\)|issue active|FP64 pipe" gpurun_out/${tag}_${k}_ncu.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/${tag}_launch_run.log 2>&1
echo "launch list rc=$?"
python tools/summarize_launches.py gpurun_out/${tag}_launches.csv "${tag} (${commit}) launch list (ncu gpu__time_duration + dram bytes, --clock-control none; bench.py --steps 2 --warmup 1; cold-cache, serialised)" > gpurun_out/${tag}_launches_summary.txt 2>&1
head -30 gpurun_out/${tag}_launches_summary.txt
(nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap \
    --format=csv -lms 200 > gpurun_out/${tag}_clocks.csv) &
smi=$!
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"
kill $smi 2>/dev/null
tail -1 gpurun_out/${tag}_bench.json | cut -c1-900
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_reference.json 2>gpurun_out/${tag}_reference.err
echo "reference rc=$?"; tail -1 gpurun_out/${tag}_reference.json | cut -c1-400
