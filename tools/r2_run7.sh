mkdir -p gpurun_out
nproc; python -c "import os; print(len(os.sched_getaffinity(0)))"
timeout 900 python -m pytest tests/test_gpu_multidevice.py -q -x --timeout 800 > gpurun_out/multidev.log 2>&1; echo "multidev rc=$?"; tail -15 gpurun_out/multidev.log
for t in 4 8 12 16 24; do echo "threads $t"; L0S_COPY_THREADS=$t timeout 300 python tools/e2e_probe.py 2>&1 | grep pageable; done
