for ich in 256 512 1024 4096; do
  echo "ich=$ich $(L0S_ICH=$ich python tools/tune_fit.py one | python -c 'import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print(d["fit_ms_min"], d["fit_ms_med"], d["total_ms"])')"
done
