timeout 900 python -m pytest tests/test_gpu_parity.py -k "ozaki or chunked or gram or incremental" -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/time_stage.py 2>&1 | tail -1 | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_oz_gemm -s 2 -c 1 --csv --log-file gpurun_out/r2u.csv python tools/time_stage.py > /dev/null 2>&1
grep -E "duration|tc_cycles" gpurun_out/r2u.csv | cut -d, -f13-16
