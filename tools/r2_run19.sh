mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/r2d_tests.log 2>&1; echo "tests rc=$?"
tail -25 gpurun_out/r2d_tests.log
timeout 600 python tools/parts_balance.py c3 8 > gpurun_out/r2d_parts_c3.json 2>&1; echo "parts rc=$?"; cut -c1-600 gpurun_out/r2d_parts_c3.json
L0S_EXACT_SPLIT=0 timeout 600 python tools/parts_balance.py c3 8 > gpurun_out/r2d_parts_c3_nosplit.json 2>&1; cut -c1-300 gpurun_out/r2d_parts_c3_nosplit.json
timeout 900 python tools/cliff_check.py > gpurun_out/r2d_cliff.jsonl 2> gpurun_out/r2d_cliff.err; echo "cliff rc=$?"; cut -c1-250 gpurun_out/r2d_cliff.jsonl; tail -3 gpurun_out/r2d_cliff.err
