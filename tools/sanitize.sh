# compute-sanitizer over the kernels (run under gpurun; one GPU).
#   bash tools/sanitize.sh <tag>
set -u
tag=${1:-r2}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 99 --print-limit 50 python tools/sanitize_probe.py \
      > gpurun_out/${tag}_sanitizer_${tool}.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/${tag}_sanitizer_${tool}.log
done
timeout 1800 $CS --tool memcheck --error-exitcode 99 --print-limit 50 python -m pytest -q -x tests/test_gpu_api.py \
    tests/test_gpu_multidevice.py "tests/test_gpu_scale.py::test_stress_loop_matches_oracle[0]" \
    > gpurun_out/${tag}_sanitizer_memcheck_tests.log 2>&1
echo "memcheck tests rc=$?"; tail -3 gpurun_out/${tag}_sanitizer_memcheck_tests.log
