mkdir -p gpurun_out
tag=${1:-r2e}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dd_screen or qr_screen or search_parts" -p no:cacheprovider > gpurun_out/${tag}_qr.log 2>&1; echo "qr tests rc=$?"; tail -25 gpurun_out/${tag}_qr.log
timeout 600 python tools/c4_once.py > gpurun_out/${tag}_c4_once.txt 2>&1; echo "c4 rc=$?"; cut -c1-900 gpurun_out/${tag}_c4_once.txt
L0S_QR_SCREEN=tsqr timeout 600 python tools/c4_once.py 2>&1 | cut -c1-300
timeout 900 python tools/run_configs.py c4 --check > gpurun_out/${tag}_configs.jsonl 2>&1; echo "configs rc=$?"; cut -c1-1200 gpurun_out/${tag}_configs.jsonl
timeout 900 python tools/parts_balance.py c4 8 > gpurun_out/${tag}_parts_c4.json 2> gpurun_out/${tag}_parts_c4.err; echo "parts rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/${tag}_parts_c4.json')); u=d['units']
print('c4 whole',d['whole_ms'],'max part',u['max_ms'],'fit',u['fit_ms'],'exact',u['exact_ms'],'cand',u['candidates'],'resc',u['rescans'])"
