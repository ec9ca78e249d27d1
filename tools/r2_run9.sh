mkdir -p gpurun_out
timeout 900 python tools/cliff_check.py > gpurun_out/cliff.jsonl 2> gpurun_out/cliff.err; echo "cliff rc=$?"; cat gpurun_out/cliff.jsonl; tail -3 gpurun_out/cliff.err
bash tools/sanitize.sh r2
