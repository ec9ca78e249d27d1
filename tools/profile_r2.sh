# Round-2 profiling captures (run under gpurun; one GPU, never multi-rank).
#   bash tools/profile_r2.sh <tag>
# 1. launch list of a short bench (device time + DRAM bytes of every launch; cold-cache, serialised)
# 2. ncu --set full (+ source) of k_fit3<4> on C3, planted y and y ~ N(0,1)
# 3. ncu --set full of the staging kernels (k_gather, k_normalize) and the INT8 Gram (k_oz_gemm)
# 4. the bench itself with nvidia-smi clocks sampled during it
set -u
tag=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/${tag}_launch_run.log 2>&1
echo "launch list rc=$?"
python tools/summarize_launches.py gpurun_out/${tag}_launches.csv "${tag} launch list (ncu gpu__time_duration + dram bytes, --clock-control none; bench.py --steps 2 --warmup 1; cold-cache, serialised)" > gpurun_out/${tag}_launches_summary.txt 2>&1
for y in planted random; do
  L0S_TUNE_Y=$y timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fit3 -s 2 -c 1 -f \
      -o gpurun_out/${tag}_fit3_${y} python tools/tune_fit.py one > gpurun_out/${tag}_fit3_${y}.log 2>&1
  echo "fit3 $y rc=$?"
  python tools/ncu_summary.py gpurun_out/${tag}_fit3_${y}.ncu-rep "${tag}: k_fit3<4> on C3, ${y} y" > gpurun_out/${tag}_fit3_${y}_ncu.txt
  ncu -i gpurun_out/${tag}_fit3_${y}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_fit3_${y}_src.csv 2>/dev/null
  python tools/ncu_blocks.py gpurun_out/${tag}_fit3_${y}_src.csv 10 > gpurun_out/${tag}_fit3_${y}_blocks.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gather|k_normalize|k_oz_gemm" -s 5 -c 5 -f \
    -o gpurun_out/${tag}_stage python tools/time_stage.py > gpurun_out/${tag}_stage.log 2>&1
echo "stage full rc=$?"
python tools/ncu_summary.py gpurun_out/${tag}_stage.ncu-rep "${tag}: staging kernels and the INT8 Gram on C3" > gpurun_out/${tag}_stage_ncu.txt
(nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap \
    --format=csv -lms 200 > gpurun_out/${tag}_clocks.csv) &
smi=$!
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"
kill $smi 2>/dev/null
tail -1 gpurun_out/${tag}_bench.json | cut -c1-600
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_reference.json 2>&1
echo "reference rc=$?"; tail -1 gpurun_out/${tag}_reference.json | cut -c1-300
