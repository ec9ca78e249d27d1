"""Golden fixtures at BASELINE scale, made by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_scale.py [--workers 8]

For C2 (600 features x 1000 samples, n = 3: every one of the 35,820,200 tuples) in both
variants of SURVEY.md 8(d) -- planted y and y ~ N(0,1) -- it runs descsearch.search.l0_search
(search.py:202-322, numba kernels) with the package's own worker threads and writes the top
10 models (indices, score, coefficients, rmse bits) to scale_c2_<variant>.npz, together with a
sha256 digest of the inputs (tests/scale_cases.py regenerates them on the GPU box).
"""

from __future__ import annotations

import argparse
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402

from descsearch import search  # noqa: E402
import scale_cases  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    for variant in ("planted", "random"):
        if args.only and variant != args.only:
            continue
        v, y, slices = scale_cases.c2(variant)
        cfg = search.L0Config(dimension=3, n_models_store=10, autotune=False)
        st = search.SearchStats()
        t0 = time.perf_counter()
        models = search.l0_search(v, y, slices, cfg, workers=args.workers, stats=st)
        dt = time.perf_counter() - t0
        out = os.path.join(HERE, f"scale_c2_{variant}.npz")
        np.savez(out, digest=scale_cases.digest(v, y), n=3, keep=10,
                 exp_indices=np.array([md.indices for md in models], dtype=np.int64),
                 exp_score=np.array([md.score for md in models]),
                 exp_coef=np.array([md.coefficients for md in models]),
                 exp_rmse=np.array([md.rmse_per_task for md in models]),
                 seconds=dt, workers=args.workers, n_tuples=st.n_tuples)
        print(variant, f"{dt:.1f} s on {args.workers} workers", models[0].indices, models[0].score, flush=True)


if __name__ == "__main__":
    main()
