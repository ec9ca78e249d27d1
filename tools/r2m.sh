timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/r2m_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2m_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2m_bench.json 2>gpurun_out/r2m_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2m_bench.json').read().strip().splitlines()[-1])
print('ms',d['ms_per_step'],'e2e',d['e2e']['value'],'fit',d['detail']['fit_ms'],'stage',d['detail']['stage_gram_ms'],d['roofline_stage'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stage_rows -s 3 -c 1 -f -o gpurun_out/r2m_stage_rows python tools/time_stage.py > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/r2m_stage_rows.ncu-rep "r2m: k_stage_rows (feature rows, integer digit extraction) on C3" > gpurun_out/r2m_stage_rows_ncu.txt
grep -E "duration|DRAM throughput|DRAM %|issue active" gpurun_out/r2m_stage_rows_ncu.txt
