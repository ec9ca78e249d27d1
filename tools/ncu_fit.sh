# ncu --set full of one screened-fit launch (C3 via tools/tune_fit.py one), with source counters.
#   bash tools/ncu_fit.sh <tag> [kernel-regex]
set -u
tag=${1:-fit}
kre=${2:-k_fit3}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${kre} -s 2 -c 1 -f \
    -o gpurun_out/${tag} python tools/tune_fit.py one > gpurun_out/${tag}.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/${tag}.ncu-rep "${tag}" > gpurun_out/${tag}_summary.txt 2>&1
cat gpurun_out/${tag}_summary.txt
