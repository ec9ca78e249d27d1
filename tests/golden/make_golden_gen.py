"""Golden fixtures for the streamed last rung, made by running the REFERENCE.

    python tests/golden/make_golden_gen.py

Imports descsearch from /root/reference/pkg/src and writes, next to this file:

* gen_<name>.npz  : generation.iter_final_rung (generation.py:331-393) over the pool the
                    pipeline builds (rungs < max_rung materialized by generate_rung): the
                    kept expressions per yielded chunk (rendered), a blake2b digest of each
                    chunk's value matrix bytes, and the RungStats counters.
* pipestream_<name>.npz : run_pipeline with materialize_last_rung=False -- the models_dim<d>.txt
                    bytes written by write_outputs (the same layout as make_golden.py's).

The GPU box never runs this script; the tests read the committed fixtures.
"""

from __future__ import annotations

import hashlib
import os
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from descsearch.dataio import RunConfig, make_synthetic_dataset  # noqa: E402
from descsearch.expressions import get_operator, render  # noqa: E402
from descsearch.generation import FeatureSpace, GenerationConfig, RungStats, generate_rung, iter_final_rung  # noqa: E402
from descsearch.pipeline import run_pipeline, write_outputs  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    # name: (dataset kwargs, operators, max_rung, precision, value_batch_size, extra limits)
    "stream_c1": (dict(n_primary=10, n_samples=100, n_tasks=1, seed=0), ["add", "sub", "mul", "div", "sqrt"], 2,
                  "fp64", 50_000, {}),
    "stream_ops": (dict(n_primary=6, n_samples=90, n_tasks=3, seed=4),
                   ["abs_diff", "sq", "cb", "inv", "abs", "exp", "log", "cbrt"], 2, "fp64", 7_000, {}),
    "stream_fp32": (dict(n_primary=7, n_samples=64, n_tasks=2, seed=7), ["add", "mul", "div", "sqrt", "sub"], 2,
                    "fp32", 100_000, dict(min_abs_value=1e-3, max_abs_value=1e3)),
}


def pool_for(ds, ops, max_rung, precision, limits):
    pool = FeatureSpace.from_primaries(ds.primary_names, ds.primary_units, ds.primary_values, precision=precision,
                                       dedup_tolerance=1e-12)
    gcfg = GenerationConfig(operators=[get_operator(o) for o in ops], max_rung=max_rung, materialize_last_rung=False,
                            **limits)
    for r in range(1, max_rung):
        generate_rung(pool, r, gcfg)
    return pool, gcfg


def record_generation(name):
    dsk, ops, max_rung, precision, vbs, limits = CASES[name]
    ds = make_synthetic_dataset(**dsk)
    pool, gcfg = pool_for(ds, ops, max_rung, precision, limits)
    gcfg.value_batch_size = vbs
    stats = RungStats(rung=max_rung)
    exprs, digests, sizes = [], [], []
    for ex, mat in iter_final_rung(pool, gcfg, 1, None, stats):
        exprs.extend(render(e) for e in ex)
        sizes.append(len(ex))
        digests.append(hashlib.blake2b(np.ascontiguousarray(mat).tobytes(), digest_size=16).hexdigest())
    arrays = {"exprs": np.array(exprs), "sizes": np.array(sizes, dtype=np.int64), "digests": np.array(digests),
              "stats": np.array([stats.n_pairs, stats.n_invalid, stats.n_dup_key, stats.n_dup_value, stats.n_kept],
                                dtype=np.int64),
              "pool_size": np.int64(len(pool))}
    np.savez_compressed(os.path.join(HERE, f"gen_{name}.npz"), **arrays)
    print(f"gen_{name}: pool {len(pool)}, pairs {stats.n_pairs}, kept {stats.n_kept}, chunks {len(sizes)}")


def record_stream_pipeline(name, dim, n_sis):
    dsk, ops, max_rung, precision, vbs, limits = CASES[name]
    ds = make_synthetic_dataset(**dsk)
    cfg = RunConfig(property_key="target", operators=ops, max_rung=max_rung, dimension=dim, n_sis_select=n_sis,
                    autotune=False, materialize_last_rung=False, precision=precision, value_batch_size=vbs,
                    **limits)
    result = run_pipeline(ds, cfg)
    files = {}
    with tempfile.TemporaryDirectory() as td:
        write_outputs(result, cfg, td)
        for d in range(1, dim + 1):
            with open(os.path.join(td, f"models_dim{d}.txt"), "rb") as fh:
                files[f"d{d}_models_file"] = np.frombuffer(fh.read(), dtype=np.uint8)
    keys = [render(e.expression) for e in result.subspace.entries]
    np.savez_compressed(os.path.join(HERE, f"pipestream_{name}.npz"), n_dims=np.int64(dim), subspace=np.array(keys),
                        **files)
    print(f"pipestream_{name}: subspace {len(keys)}")


def main():
    for name in CASES:
        record_generation(name)
    record_stream_pipeline("stream_c1", 2, 20)
    record_stream_pipeline("stream_ops", 2, 15)
    record_stream_pipeline("stream_fp32", 2, 12)


if __name__ == "__main__":
    main()
