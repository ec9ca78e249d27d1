# C4 (dim 4) with each tune_fit variant library, screened and plain sweeps
for v in ${VARIANTS:-base}; do
  for scr in 1 0; do
    echo "== $v screen=$scr"
    L0S_TILE_SCREEN=$scr L0S_LIB=$PWD/paper_2502_20072_b200/variants/lib_$v.so timeout 600 python tools/run_configs.py c4 2>&1 | cut -c1-260
  done
done
