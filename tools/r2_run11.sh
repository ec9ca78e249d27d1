mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
( time timeout 1800 python -m pytest tests -m gpu -q -x --timeout 1500 -p no:cacheprovider ) > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -8 gpurun_out/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
bash tools/profile_r2.sh r2a
