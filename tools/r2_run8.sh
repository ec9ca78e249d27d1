mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -25 gpurun_out/gpu_tests.log
timeout 600 python tools/cliff_check.py > gpurun_out/cliff.jsonl 2> gpurun_out/cliff.err; echo "cliff rc=$?"; cat gpurun_out/cliff.jsonl; tail -3 gpurun_out/cliff.err
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.txt 2>&1; echo "e2e rc=$?"; grep -E "pageable|Register" gpurun_out/e2e_probe.txt
