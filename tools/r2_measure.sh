# round-2 measurements for DESIGN.md / profiles (tag = $1): emulated multi-GPU parts, cliff
# shapes, end-to-end phases, staging + Gram ncu captures
tag=${1:-r2m}
mkdir -p gpurun_out
for c in c3 c4; do
  timeout 900 python tools/parts_balance.py $c 8 > gpurun_out/${tag}_parts_$c.json 2> gpurun_out/${tag}_parts_$c.err; echo "parts $c rc=$?"
  cut -c1-400 gpurun_out/${tag}_parts_$c.json
done
timeout 900 python tools/cliff_check.py > gpurun_out/${tag}_cliff.jsonl 2> gpurun_out/${tag}_cliff.err; echo "cliff rc=$?"
cut -c1-200 gpurun_out/${tag}_cliff.jsonl
timeout 300 python tools/e2e_probe.py > gpurun_out/${tag}_e2e_probe.txt 2>&1; echo "e2e rc=$?"; tail -8 gpurun_out/${tag}_e2e_probe.txt
for k in k_gather k_normalize k_oz_gemm; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -f \
      -o gpurun_out/${tag}_$k python tools/time_stage.py > gpurun_out/${tag}_$k.log 2>&1
  echo "ncu $k rc=$?"
  python tools/ncu_summary.py gpurun_out/${tag}_$k.ncu-rep "${tag}: $k on C3" > gpurun_out/${tag}_${k}_ncu.txt
  grep -E "duration|DRAM (read|write)|DRAM throughput|grid|issue active|tensor" gpurun_out/${tag}_${k}_ncu.txt
done
