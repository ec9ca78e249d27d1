mkdir -p gpurun_out
gcc -O3 -mavx2 -pthread tools/micro/hostbw.c -o /tmp/hostbw && /tmp/hostbw > gpurun_out/hostbw.txt; cat gpurun_out/hostbw.txt
nproc; lscpu | grep -E "Model name|Socket|NUMA node|Thread|Core"
python - <<'P'
import json,sys
sys.path.insert(0,'.')
import numpy as np, torch
import bench
from paper_2502_20072_b200 import _lib
from paper_2502_20072_b200.search import _partition
v,y,sl=bench.make_c3(); perm,bounds,_=_partition(bench.S,sl)
eng=_lib.engine(0)
vd,yd,pd=(torch.from_numpy(x).cuda() for x in (v,y,perm))
ts=[]
for _ in range(6):
    eng.stage((bench.M,bench.S),None,None,bounds,"fp64",device_ptrs=(vd.data_ptr(),yd.data_ptr(),pd.data_ptr()))
    ts.append(eng.stage_timings())
print(ts[-1])
P
for th in 8 16; do L0S_COPY_THREADS=$th timeout 300 python tools/e2e_probe.py 2>&1 | grep pageable | tail -2 | sed "s/^/threads $th: /"; done
