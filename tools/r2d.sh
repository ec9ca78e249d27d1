mkdir -p gpurun_out
tag=${1:-r2d}
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${tag}_tests.log
for c in c3 c4; do
  timeout 900 python tools/parts_balance.py $c 8 > gpurun_out/${tag}_parts_$c.json 2> gpurun_out/${tag}_parts_$c.err; echo "parts $c rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/${tag}_parts_$c.json')); u=d['units']
print('$c whole',d['whole_ms'],'max part',u['max_ms'],'fit',u['fit_ms'],'exact',u['exact_ms'],'cand',u['candidates'],'resc',u['rescans'])"
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench.json 2>gpurun_out/${tag}_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/${tag}_bench.json').read().strip().splitlines()[-1])
print('ms',d['ms_per_step'],'e2e',d['e2e']['value'],'fit',d['detail']['fit_ms'],'exact',d['detail']['exact_ms'],'cand',d['detail']['n_candidates']); r=d['random_y']; print('random ms',r['ms_per_step'],'fit',r['fit_ms'],r['gram'])"
