for c in c3 c4; do for n in 2 4 8; do
  timeout 900 python tools/parts_balance.py $c $n > gpurun_out/r2w_parts_${c}_$n.json 2> gpurun_out/r2w_parts_${c}_$n.err
  python -c "
import json; d=json.load(open('gpurun_out/r2w_parts_${c}_$n.json'))
u=d['units_exchange']; print('$c', $n, 'whole', round(d['whole_ms'],3), 'max part', round(u['max_ms'],3), 'mean', round(u['mean_ms'],3), 'rescans', sum(u['rescans']))"
done; done
timeout 300 python tools/time_stage.py 2>&1 | tail -1 | cut -c1-100
python - <<'PY'
import sys, json; sys.path.insert(0, '.')
from tools.run_configs import make_c4
from paper_2502_20072_b200 import _lib
from paper_2502_20072_b200.search import _partition
v, y, sl, n = make_c4(); perm, b, _ = _partition(v.shape[1], sl); e = _lib.engine(0)
for _ in range(3): e.stage(v, y, perm, b, "fp64")
import torch
vd, yd, pd = (torch.from_numpy(x).cuda() for x in (v, y, perm)); ms = []
for _ in range(5):
    e.stage(v.shape, None, None, b, "fp64", device_ptrs=(vd.data_ptr(), yd.data_ptr(), pd.data_ptr())); sc, rk, *_r, st = e.search(4, 10, 0, 2**62, "fast"); ms.append(st.ms_gram)
print("c4 stage ms", sorted(ms)[2])
PY
