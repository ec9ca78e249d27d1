timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/r2x_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2x_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2x_bench.json 2>gpurun_out/r2x_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2x_bench.json').read().strip().splitlines()[-1])
print('ms',d['ms_per_step'],'e2e',d['e2e']['value'],'fit',d['detail']['fit_ms'],'stage',d['detail']['stage_gram_ms'],'search',d['detail']['search_ms'],'exact',d['detail']['exact_ms'])"
timeout 600 python tools/run_configs.py c2 > gpurun_out/r2x_c2.jsonl 2>&1; cut -c1-300 gpurun_out/r2x_c2.jsonl
