# tests + bench + one ncu capture of the C3 fit kernel (tag = $1)
tag=${1:-chk}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/${tag}_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
python -c "
import json,sys; d=json.loads(open('gpurun_out/${tag}_bench.json').read().strip().splitlines()[-1])
print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'],'fit',d['detail']['fit_ms'],'random',d.get('random_y',{}).get('ms_per_step'))"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fit3 -s 2 -c 1 -f \
    -o gpurun_out/${tag}_fit3 python tools/tune_fit.py one > gpurun_out/${tag}_fit3.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/${tag}_fit3.ncu-rep "${tag}: k_fit3<4> on C3, planted y" > gpurun_out/${tag}_fit3_ncu.txt
ncu -i gpurun_out/${tag}_fit3.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_fit3_src.csv 2>/dev/null
python tools/ncu_blocks.py gpurun_out/${tag}_fit3_src.csv 12 > gpurun_out/${tag}_fit3_blocks.txt 2>&1
grep -E "duration|FP64 pipe|occupancy|issue active|stall" gpurun_out/${tag}_fit3_ncu.txt
