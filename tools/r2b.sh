set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ozaki" -p no:cacheprovider > gpurun_out/r2b_ozaki.log 2>&1; echo "ozaki tests rc=$?"; tail -15 gpurun_out/r2b_ozaki.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench.json 2>gpurun_out/r2b_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2b_bench.json').read().strip().splitlines()[-1])
print('ms',d['ms_per_step'],'e2e',d['e2e']['value'],'fit',d['detail']['fit_ms']); print(d['random_y'])"
