timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/r2v_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2v_tests.log
for v in 0 1; do if [ $v = 1 ]; then export L0S_STAGE_PER_TASK=1; fi; timeout 300 python tools/time_stage.py 2>&1 | tail -1 | cut -c1-120; python -c "
import sys; sys.path.insert(0,'.')
import torch, bench
from paper_2502_20072_b200 import _lib
from paper_2502_20072_b200.search import _partition
v,y,sl=bench.make_c3(); perm,b,_=_partition(bench.S,sl); e=_lib.engine(0)
vd,yd,pd=(torch.from_numpy(x).cuda() for x in (v,y,perm)); ms=[]
for _ in range(10):
    e.stage((bench.M,bench.S),None,None,b,'fp64',device_ptrs=(vd.data_ptr(),yd.data_ptr(),pd.data_ptr())); ms.append(e.stage_timings()['gather'])
print('per_task' if $v else 'rows', sorted(ms)[5])"; done
