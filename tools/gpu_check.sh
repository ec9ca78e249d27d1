# usage: bash tools/gpu_check.sh [tests] [bench] [ncu] [full]
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
for what in "$@"; do
case $what in
tests)
  timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
  timeout 1200 python -m pytest tests -m gpu -q --timeout 900 --durations=8 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
  grep -E "passed|failed|Error|FAILED|s call|s setup" gpurun_out/gpu_tests.log | tail -15 ;;
bench)
  timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/bench.log ;;
ncu)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
     python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu-launch rc=$?" ;;
full)
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fit3 -s 1 -c 1 -f -o gpurun_out/fit3 \
     python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"; tail -3 gpurun_out/ncu_full.log ;;
esac
done
