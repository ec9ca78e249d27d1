timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/r2l_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2l_tests.log
for c in c3 c4; do
  timeout 900 python tools/parts_balance.py $c 8 > gpurun_out/r2l_parts_$c.json 2> gpurun_out/r2l_parts_$c.err; echo "parts $c rc=$?"; tail -2 gpurun_out/r2l_parts_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/r2l_parts_$c.json'))
for k in ('units_exchange','units'):
    u=d[k]; print('$c',k,'whole',round(d['whole_ms'],2),'max part',round(u['max_ms'],2),'fit',u['fit_ms'],'exact',u['exact_ms'],'cand',u['candidates'],'resc',u['rescans'])"
done
