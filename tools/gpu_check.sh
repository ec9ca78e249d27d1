mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -5 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 8 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -5 gpurun_out/bench.log
