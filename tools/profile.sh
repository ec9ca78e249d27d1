# Profiling captures for profiles/ (run under gpurun; one GPU, never multi-rank).
#   bash tools/profile.sh <tag>
# 1. launch list of a short bench (device time of every launch; cold-cache, serialised)
# 2. ncu --set full of the screened fit kernel and of one Gram launch
# 3. clocks during a normal bench run
set -u
tag=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/${tag}_launch_run.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fit3 -s 2 -c 1 -f \
    -o gpurun_out/${tag}_fit3 python tools/tune_fit.py one > gpurun_out/${tag}_fit3.log 2>&1
echo "fit3 full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_oz_gemm -s 1 -c 1 -f \
    -o gpurun_out/${tag}_gram python tools/time_stage.py > gpurun_out/${tag}_gram.log 2>&1
echo "gram full rc=$?"
(nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap \
    --format=csv -lms 200 > gpurun_out/${tag}_clocks.csv) &
smi=$!
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"
kill $smi 2>/dev/null
tail -1 gpurun_out/${tag}_bench.json
python tools/summarize_launches.py gpurun_out/${tag}_launches.csv "${tag} launch list (ncu gpu__time_duration + dram bytes, --clock-control none; bench.py --steps 2 --warmup 1; cold-cache, serialised)" > gpurun_out/${tag}_launches_summary.txt
timeout 300 python tools/e2e_probe.py > gpurun_out/${tag}_e2e_probe.txt 2>&1
echo "e2e probe rc=$?"
