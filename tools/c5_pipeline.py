"""BASELINE C5 with real feature generation: run_pipeline (drop-in installed) with the last
rung streamed through the device -- candidate values, validity and fingerprints
(csrc/gen.cu), SIS scores (csrc/sis.cu), the screen, the dim-1..3 l0 searches.

    python tools/c5_pipeline.py [--primaries 24] [--samples 2000] [--select 200]

Prints one JSON line: candidates per dimension, wall time per phase, the reference's
single-core generation rate on a bounded sample (tools/gen_bench.py's method) for scale.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
if os.path.isdir(ref):
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_l0s")
    sys.path.append(ref)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--primaries", type=int, default=24)
    ap.add_argument("--samples", type=int, default=2000)
    ap.add_argument("--select", type=int, default=200)
    ap.add_argument("--dimension", type=int, default=3)
    args = ap.parse_args()
    from descsearch.dataio import RunConfig, make_synthetic_dataset
    from descsearch.pipeline import run_pipeline

    import paper_2502_20072_b200 as l0

    ds = make_synthetic_dataset(n_primary=args.primaries, n_samples=args.samples, n_tasks=1, seed=5)
    cfg = RunConfig(property_key="target", operators=["add", "sub", "mul", "div", "sqrt"], max_rung=2,
                    dimension=args.dimension, n_sis_select=args.select, autotune=False,
                    materialize_last_rung=False, value_batch_size=1_000_000)
    undo = l0.install()
    try:
        t0 = time.perf_counter()
        res = run_pipeline(ds, cfg)
        wall = time.perf_counter() - t0
    finally:
        undo()
    t = res.timings
    out = {"primaries": args.primaries, "samples": args.samples, "n_sis_select": args.select,
           "wall_s": wall, "feature_generation_s": t.feature_generation, "screening_s": t.screening,
           "descriptor_search_s": t.descriptor_search,
           "pool_size": res.pool_size, "rung_stats": [vars(r) for r in res.rung_stats],
           "dims": [{"d": d.dimension, "subspace": d.subspace_size, "tuples": d.search_stats.n_tuples,
                     "best": [str(e) for e in d.models[0].expressions] if d.models[0].expressions else None,
                     "score": d.models[0].score} for d in res.dimensions]}
    print(json.dumps(out, default=str))


if __name__ == "__main__":
    main()
