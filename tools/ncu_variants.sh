# ncu --set full of k_fit3 for each tune_fit variant (planted y unless L0S_TUNE_Y), one capture each
mkdir -p gpurun_out
for v in ${VARIANTS:-base no_tile_screen}; do
  L0S_LIB=paper_2502_20072_b200/variants/lib_$v.so timeout 900 ncu --set full --clock-control none --import-source on \
      --kernel-name-base demangled -k "regex:k_fit3.*bool.1" -s 1 -c 1 -f -o gpurun_out/var_$v python tools/tune_fit.py one > gpurun_out/var_$v.log 2>&1
  python tools/ncu_summary.py gpurun_out/var_$v.ncu-rep "$v" > gpurun_out/var_${v}_ncu.txt
  cat gpurun_out/var_${v}_ncu.txt
done
