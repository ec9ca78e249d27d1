tag=${1:-r2k}
mkdir -p gpurun_out
timeout 300 python tools/sanitize_probe.py; echo "probe rc=$?"
bash tools/sanitize.sh $tag
timeout 900 python tools/cliff_check.py > gpurun_out/${tag}_cliff.jsonl 2> gpurun_out/${tag}_cliff.err; echo "cliff rc=$?"; cut -c1-220 gpurun_out/${tag}_cliff.jsonl
timeout 900 python tools/run_configs.py c2 c4 --check > gpurun_out/${tag}_configs.jsonl 2>&1; echo "configs rc=$?"; cut -c1-300 gpurun_out/${tag}_configs.jsonl
