"""cProfile of the C5 pipeline (tools/c5_pipeline.py's run): where the host time goes."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
if os.path.isdir(ref):
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_l0s")
    sys.path.append(ref)
from descsearch.dataio import RunConfig, make_synthetic_dataset  # noqa: E402
from descsearch.pipeline import run_pipeline  # noqa: E402

import paper_2502_20072_b200 as l0  # noqa: E402

ds = make_synthetic_dataset(n_primary=24, n_samples=2000, n_tasks=1, seed=5)
cfg = RunConfig(property_key="target", operators=["add", "sub", "mul", "div", "sqrt"], max_rung=2, dimension=3,
                n_sis_select=200, autotune=False, materialize_last_rung=False, value_batch_size=1_000_000)
undo = l0.install()
run_pipeline(ds, cfg)  # warm
pr = cProfile.Profile()
pr.enable()
res = run_pipeline(ds, cfg)
pr.disable()
undo()
print(vars(res.timings))
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(30)
