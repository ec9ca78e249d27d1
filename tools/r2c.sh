# round-2 measurements: emulated multi-GPU parts (C3, C4), other configs, C4 breakdown, e2e phases,
# ncu of the feature-row staging kernel (tag = $1)
tag=${1:-r2c}
mkdir -p gpurun_out
for c in c3 c4; do
  timeout 900 python tools/parts_balance.py $c 8 > gpurun_out/${tag}_parts_$c.json 2> gpurun_out/${tag}_parts_$c.err; echo "parts $c rc=$?"
  cut -c1-700 gpurun_out/${tag}_parts_$c.json
done
timeout 900 python tools/run_configs.py c2 c4 --check > gpurun_out/${tag}_configs.jsonl 2>&1; echo "configs rc=$?"; cut -c1-400 gpurun_out/${tag}_configs.jsonl
timeout 300 python tools/c4_once.py > gpurun_out/${tag}_c4_once.txt 2>&1; echo "c4 rc=$?"; cut -c1-1500 gpurun_out/${tag}_c4_once.txt
timeout 300 python tools/e2e_probe.py > gpurun_out/${tag}_e2e_probe.txt 2>&1; echo "e2e rc=$?"; tail -12 gpurun_out/${tag}_e2e_probe.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stage_rows -s 3 -c 1 -f \
    -o gpurun_out/${tag}_stage_rows python tools/time_stage.py > gpurun_out/${tag}_stage_rows.log 2>&1
echo "ncu stage_rows rc=$?"
python tools/ncu_summary.py gpurun_out/${tag}_stage_rows.ncu-rep "${tag}: k_stage_rows (feature rows) on C3" > gpurun_out/${tag}_stage_rows_ncu.txt
grep -E "grid|duration|DRAM (read|write)|DRAM throughput|DRAM %|issue active" gpurun_out/${tag}_stage_rows_ncu.txt
