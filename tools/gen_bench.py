"""Streamed last rung: candidates/s of the device path vs the reference (run under gpurun).

    python tools/gen_bench.py [--primaries 14] [--samples 2000] [--ops add,sub,mul,div,sqrt]

Pool = primaries + rung 1 (the reference's generate_rung), last rung (2) streamed.  Times
the reference's iter_final_rung (numpy, 1 thread) on the first --ref-pairs candidates of the
first operator, and this package's iter_final_rung (host matrices, and DeviceChunk blocks)
plus sis_select over the device stream on the whole rung.  One JSON line.
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

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--primaries", type=int, default=14)
    ap.add_argument("--samples", type=int, default=2000)
    ap.add_argument("--ops", default="add,sub,mul,div,sqrt")
    ap.add_argument("--ref-pairs", type=int, default=20000)
    args = ap.parse_args()
    from descsearch.dataio import make_synthetic_dataset
    from descsearch.expressions import get_operator
    from descsearch.generation import FeatureSpace, GenerationConfig, RungStats, generate_rung
    from descsearch.generation import iter_final_rung as ref_iter
    from descsearch.screening import ScreeningTarget

    from paper_2502_20072_b200.generation import iter_final_rung
    from paper_2502_20072_b200.screening import sis_select

    ds = make_synthetic_dataset(n_primary=args.primaries, n_samples=args.samples, n_tasks=1, seed=0)
    ops = [get_operator(o) for o in args.ops.split(",")]
    pool = FeatureSpace.from_primaries(ds.primary_names, ds.primary_units, ds.primary_values)
    gcfg = GenerationConfig(operators=ops, max_rung=2, materialize_last_rung=False, value_batch_size=1_000_000)
    generate_rung(pool, 1, gcfg)
    out = {"pool": len(pool), "samples": args.samples, "ops": args.ops}
    # reference: a bounded sample (first operator only)
    g1 = GenerationConfig(operators=ops[:1], max_rung=2, materialize_last_rung=False,
                          value_batch_size=args.ref_pairs)
    st = RungStats(rung=2)
    t0 = time.perf_counter()
    it = ref_iter(pool, g1, 1, None, st)
    next(it)
    t_ref = time.perf_counter() - t0
    out["ref_sample_pairs"] = args.ref_pairs
    out["ref_cand_per_s"] = args.ref_pairs / t_ref
    for _ in range(2):  # warm-up + timed
        st = RungStats(rung=2)
        t0 = time.perf_counter()
        n = sum(len(ex) for ex, _ in iter_final_rung(pool, gcfg, 1, None, st))
        t_host = time.perf_counter() - t0
    out["pairs"] = st.n_pairs
    out["kept"] = n
    out["host_matrices_cand_per_s"] = st.n_pairs / t_host
    st = RungStats(rung=2)
    t0 = time.perf_counter()
    n = sum(len(ex) for ex, _ in iter_final_rung(pool, gcfg, 1, None, st, on_device=True))
    out["device_chunks_cand_per_s"] = st.n_pairs / (time.perf_counter() - t0)
    labels, slices = ds.task_partition()
    y = np.asarray(ds.property_values, dtype=np.float64)
    target = ScreeningTarget([y], slices, labels)
    t0 = time.perf_counter()
    sub = sis_select(iter_final_rung(pool, gcfg, on_device=True), target, 200)
    out["stream_plus_sis_cand_per_s"] = st.n_pairs / (time.perf_counter() - t0)
    out["selected"] = len(sub)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
