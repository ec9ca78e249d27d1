for w in planted random mt4; do timeout 900 python tools/c4_var.py $w 3 2>&1 | tail -2; done
timeout 900 python tools/parts_balance.py c4 8 > gpurun_out/r2i_parts_c4.json 2> gpurun_out/r2i_parts_c4.err; echo "parts rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r2i_parts_c4.json')); u=d['units']
print('c4 whole',d['whole_ms'],'max part',u['max_ms'],'fit',u['fit_ms'],'exact',u['exact_ms'],'cand',u['candidates'],'resc',u['rescans'])"
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/r2i_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2i_tests.log
