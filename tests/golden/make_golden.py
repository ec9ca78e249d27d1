"""Generate the golden parity fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports descsearch from /root/reference/pkg/src (numba kernels, lsq.py and
search.py) and writes small .npz fixtures next to this file.  The GPU box
never runs this script; the tests read the committed fixtures.

Fixture kinds
-------------
* lsq_<name>.npz    : score_tuples (lsq.py:113-156) over every tuple of a small
                      instance, plus fit_tuple_kernel (lsq.py:159-192) outputs
                      for a sample of tuples -- exact float bits.
* search_<name>.npz : l0_search (search.py:202-322) results -- indices, score,
                      coefficients, rmse_per_task (exact bits), plus the
                      instance (values, y, task ids, dimension, keep, precision).
* pipe_<name>.npz   : the inputs l0_search received inside run_pipeline
                      (pipeline.py:219-229) for every dimension, the models it
                      returned, and the models_dim<d>.txt bytes written by
                      write_outputs.
"""

from __future__ import annotations

import itertools
import os
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import descsearch  # noqa: E402
from descsearch import lsq, search  # noqa: E402
from descsearch.dataio import RunConfig, make_synthetic_dataset, Dataset  # noqa: E402
from descsearch.expressions import render  # noqa: E402
from descsearch.pipeline import run_pipeline, write_outputs  # noqa: E402
from descsearch.units import Unit  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def _task_ids(slices, s):
    tid = np.full(s, -1, dtype=np.int64)
    order = np.concatenate([np.asarray(sl) for sl in slices])
    for t, sl in enumerate(slices):
        tid[np.asarray(sl)] = t
    return tid, order


def slices_from(task_id, order):
    """Inverse of _task_ids: slices in task order, each in the recorded order."""
    out = []
    for t in range(int(task_id.max()) + 1):
        out.append(np.array([i for i in order if task_id[i] == t], dtype=np.int64))
    return out


def models_arrays(models, T, n):
    k = len(models)
    idx = np.zeros((k, n), dtype=np.int64)
    score = np.zeros(k)
    coef = np.zeros((k, T, n + 1))
    rmse = np.zeros((k, T))
    for i, md in enumerate(models):
        idx[i] = md.indices
        score[i] = md.score
        coef[i] = md.coefficients
        rmse[i] = md.rmse_per_task
    return idx, score, coef, rmse


def save_search(name, values, y, slices, n, keep=10, precision="fp64", all_scores=True, labels=None):
    values = np.asarray(values, dtype=np.float64)
    s = values.shape[1]
    if slices is None:
        slices = [np.arange(s)]
    cfg = search.L0Config(dimension=n, autotune=False, n_models_store=keep, precision=precision)
    models = search.l0_search(values, y, slices, cfg, task_labels=labels)
    T = len(slices)
    idx, score, coef, rmse = models_arrays(models, T, n)
    tid, order = _task_ids(slices, s)
    extra = {}
    m = values.shape[0]
    if all_scores and search.count_models(m, n) <= 400_000:
        vals, yy, bounds, _ = search._prepare(values, y, slices, precision)
        tup = np.array(list(itertools.combinations(range(m), n)), dtype=np.int64)
        out = np.empty(len(tup), dtype=np.float64)
        lsq.score_tuples(vals, yy, bounds, tup, lsq.RANK_TOL_FACTOR[precision], out)
        extra["all_scores"] = out
    np.savez_compressed(
        os.path.join(HERE, f"search_{name}.npz"),
        values=values, y=np.asarray(y, dtype=np.float64), task_id=tid, order=order,
        n=np.int64(n), keep=np.int64(keep), precision=np.array(precision),
        exp_indices=idx, exp_score=score, exp_coef=coef, exp_rmse=rmse, **extra,
    )
    print(f"search_{name}: m={m} s={s} T={T} n={n} -> {len(models)} models")


def save_lsq(name, values, y, bounds, n, precision, rng, n_fit=64):
    dtype = np.float32 if precision == "fp32" else np.float64
    vals = np.ascontiguousarray(values, dtype=dtype)
    yy = np.ascontiguousarray(y, dtype=dtype)
    bounds = np.asarray(bounds, dtype=np.int64)
    m = vals.shape[0]
    tup = np.array(list(itertools.combinations(range(m), n)), dtype=np.int64)
    tol = lsq.RANK_TOL_FACTOR[precision]
    out = np.empty(len(tup), dtype=np.float64)
    lsq.score_tuples(vals, yy, bounds, tup, tol, out)
    pick = rng.choice(len(tup), size=min(n_fit, len(tup)), replace=False)
    T = len(bounds) - 1
    fit_ok = np.zeros(len(pick), dtype=np.int8)
    fit_coef = np.zeros((len(pick), T, n + 1), dtype=dtype)
    fit_ssr = np.zeros((len(pick), T))
    for i, t in enumerate(pick):
        c = np.zeros((T, n + 1), dtype=dtype)
        sr = np.zeros(T)
        ok = lsq.fit_tuple_kernel(vals, yy, bounds, tup[t], tol, c, sr)
        fit_ok[i] = ok
        if ok:
            fit_coef[i] = c
            fit_ssr[i] = sr
    np.savez_compressed(
        os.path.join(HERE, f"lsq_{name}.npz"),
        values=vals, y=yy, bounds=bounds, n=np.int64(n), precision=np.array(precision),
        tuples=tup, scores=out, fit_pick=pick, fit_ok=fit_ok, fit_coef=fit_coef, fit_ssr=fit_ssr,
    )
    print(f"lsq_{name}: {len(tup)} tuples, {np.isinf(out).sum()} inf, {np.isnan(out).sum()} nan")


def collinear_instance(rng, m=30, s=200, n_tasks=1):
    """Near-copies spanning the 1e-10 rank rule, near-constants, a duplicate,
    and a planted y that puts near-collinear tuples among the best ones."""
    v = rng.uniform(0.5, 2.0, size=(m, s))
    deltas = [1e-4, 1e-6, 1e-8, 1e-9, 1e-10, 1e-12]
    for i, d in enumerate(deltas):
        v[10 + i] = v[0] + d * rng.standard_normal(s)
    v[16] = 1.3 + 1e-6 * rng.standard_normal(s)
    v[17] = 0.7 + 1e-9 * rng.standard_normal(s)
    v[18] = 2.0 + 1e-12 * rng.standard_normal(s)
    v[19] = v[5]
    y = v[0] + 0.5 * v[5] + 1e-3 * rng.standard_normal(s)
    return v, y


def main():
    rng = np.random.default_rng(20260822)

    # ---- lsq (score_tuples / fit_tuple_kernel) bitwise pins ----
    v = rng.uniform(0.5, 2.0, size=(12, 30)); y = rng.standard_normal(30)
    save_lsq("rand_n2", v, y, [0, 30], 2, "fp64", rng)
    v = rng.uniform(0.5, 2.0, size=(9, 41)); y = rng.standard_normal(41)
    save_lsq("rand_n3_mt", v, y, [0, 10, 25, 41], 3, "fp64", rng)
    v = rng.uniform(0.5, 2.0, size=(8, 25)); y = rng.standard_normal(25)
    save_lsq("rand_n2_fp32", v, y, [0, 25], 2, "fp32", rng)
    v = rng.uniform(0.5, 2.0, size=(8, 33)); y = rng.standard_normal(33)
    save_lsq("rand_n3_fp32_mt", v, y, [0, 13, 33], 3, "fp32", rng)
    v, y = collinear_instance(rng, m=22, s=60)
    save_lsq("collinear_n3", v, y, [0, 60], 3, "fp64", rng, n_fit=128)
    v = rng.uniform(0.5, 2.0, size=(6, 23)); y = rng.standard_normal(23)
    v[4] = 4.25; v[3, :] = 0.0
    save_lsq("edge_rows", v, y, [0, 3, 5, 23], 2, "fp64", rng)  # rows==p, rows<p tasks
    v = rng.uniform(0.5, 2.0, size=(7, 20)); y = rng.standard_normal(20)
    v[2, 4] = np.nan; v[5, 1] = np.inf
    save_lsq("nonfinite", v, y, [0, 20], 2, "fp64", rng)
    v = rng.uniform(0.5, 2.0, size=(10, 40)) * np.logspace(-6, 6, 10)[:, None]
    y = rng.standard_normal(40)
    save_lsq("scales_n3", v, y, [0, 40], 3, "fp64", rng)

    # ---- l0_search (search.py) pins: test_search.py-style instances ----
    for n in (1, 2, 3):
        v = rng.uniform(0.5, 2.0, size=(8, 20)); y = rng.standard_normal(20)
        save_search(f"bf_n{n}", v, y, None, n)
    v = rng.uniform(0.5, 2.0, size=(7, 22)); y = rng.standard_normal(22)
    save_search("multitask", v, y, [np.arange(0, 9), np.arange(9, 22)], 2)
    v = rng.uniform(0.5, 2.0, size=(3, 15)); v[2] = v[1]; y = rng.standard_normal(15)
    save_search("tie", v, y, None, 2, keep=5)
    v = rng.uniform(0.5, 2.0, size=(2, 10)); v[1] = v[0]; y = rng.standard_normal(10)
    save_search("all_deficient", v, y, None, 2)
    v = rng.uniform(0.5, 2.0, size=(6, 25)); y = rng.standard_normal(25)
    save_search("fp32", v, y, None, 2, precision="fp32")
    v = rng.uniform(0.5, 2.0, size=(40, 300)); y = rng.standard_normal(300)
    rr = [np.arange(t, 300, 3) for t in range(3)]
    save_search("rand_mt3_n3", v, y, rr, 3)
    v = rng.uniform(0.5, 2.0, size=(30, 120))
    y = 2.0 * v[3] - 1.5 * v[17] + 0.25 * v[22] + 0.75
    save_search("planted_noiseless_n3", v, y, None, 3)
    v = rng.uniform(0.5, 2.0, size=(35, 150))
    y = 2.0 * v[3] - 1.0 * v[11] + 0.5 * v[29] + 0.5 * v[30] + 0.01 * rng.standard_normal(150)
    save_search("planted_n4", v, y, None, 4, keep=12)
    v, y = collinear_instance(rng, m=30, s=200)
    save_search("collinear_n3", v, y, None, 3, keep=20)
    v, y = collinear_instance(rng, m=24, s=90)
    save_search("collinear_n4", v, y, None, 4, keep=15)
    v = 1000.0 + rng.uniform(0.0, 1.0, size=(20, 100)); y = rng.standard_normal(100) + 50.0
    save_search("large_mean_n3", v, y, None, 3)
    v = rng.uniform(0.5, 2.0, size=(16, 60)) * np.logspace(-8, 8, 16)[:, None]
    y = rng.standard_normal(60)
    save_search("scales_n3", v, y, None, 3)
    v = rng.uniform(0.5, 2.0, size=(6, 23)); y = rng.standard_normal(23)
    save_search("rows_eq_p", v, y, [np.arange(0, 3), np.arange(3, 23)], 2)
    v = rng.uniform(0.5, 2.0, size=(7, 20)); y = rng.standard_normal(20)
    v[2, 4] = np.nan
    save_search("nan_feature", v, y, None, 2)
    v = rng.uniform(0.5, 2.0, size=(25, 64)); y = rng.standard_normal(64)
    rr = [np.arange(t, 64, 8) for t in range(8)]
    save_search("eight_tasks_n2", v, y, rr, 2)
    v = rng.uniform(0.5, 2.0, size=(14, 30)); y = rng.standard_normal(30)
    save_search("n5", v, y, None, 5, keep=7)

    # ---- run_pipeline goldens: what l0_search saw and returned, plus model files ----
    c1 = make_synthetic_dataset(n_primary=10, n_samples=100, n_tasks=1, seed=0)
    c1cfg = dict(property_key="target", operators=["add", "sub", "mul", "div", "sqrt"], max_rung=1,
                 dimension=2, n_sis_select=20, autotune=False)
    record_pipeline("c1", c1, c1cfg)
    c1mt = make_synthetic_dataset(n_primary=6, n_samples=90, n_tasks=3, seed=4)
    record_pipeline("c1_tasks3", c1mt, dict(c1cfg, dimension=3, n_sis_select=15))
    prng = np.random.default_rng(0)
    x = prng.uniform(0.5, 2.0, size=(80, 6))
    yp = 2.5 * (x[:, 1] * x[:, 2]) - 1.25 * np.sqrt(x[:, 3]) + 0.75
    names = [f"x{i}" for i in range(6)]
    planted = Dataset(sample_ids=[f"s{i}" for i in range(80)], primary_names=names,
                      primary_units=[Unit() for _ in names], primary_values=x, property_name="target",
                      property_unit=Unit(), property_values=yp, task_labels=None)
    record_pipeline("criterion3", planted, dict(property_key="target", operators=["mul", "sqrt"], max_rung=2,
                                                dimension=2, n_sis_select=300, autotune=False))


def record_pipeline(name, ds, cfgmap):
    import descsearch.pipeline as pl

    calls = []
    real = pl.l0_search

    def spy(subspace, y, slices, cfg, workers=1, task_labels=None, stats=None):
        models = real(subspace, y, slices, cfg, workers=workers, task_labels=task_labels, stats=stats)
        calls.append((subspace.values_matrix().copy(), np.asarray(y).copy(), [np.asarray(s) for s in slices],
                      cfg, tuple(task_labels), models, [render(e) for e in subspace.expressions]))
        return models

    pl.l0_search = spy
    try:
        cfg = RunConfig(**cfgmap)
        result = run_pipeline(ds, cfg)
        with tempfile.TemporaryDirectory() as td:
            write_outputs(result, cfg, td)
            files = {}
            for d in range(1, cfg.dimension + 1):
                with open(os.path.join(td, f"models_dim{d}.txt"), "rb") as fh:
                    files[d] = fh.read()
    finally:
        pl.l0_search = real
    arrays = {"n_dims": np.int64(len(calls)), "labels": np.array(calls[0][4]),
              "precision": np.array(cfg.precision), "keep": np.int64(cfg.n_models_store)}
    for d, (vals, y, slices, l0cfg, labels, models, terms) in enumerate(calls, start=1):
        T = len(slices)
        tid, order = _task_ids(slices, vals.shape[1])
        idx, score, coef, rmse = models_arrays(models, T, d)
        arrays.update({
            f"d{d}_values": vals, f"d{d}_y": y, f"d{d}_task_id": tid, f"d{d}_order": order,
            f"d{d}_terms": np.array(terms), f"d{d}_exp_indices": idx, f"d{d}_exp_score": score,
            f"d{d}_exp_coef": coef, f"d{d}_exp_rmse": rmse,
            f"d{d}_models_file": np.frombuffer(files[d], dtype=np.uint8),
        })
        print(f"pipe_{name} d={d}: m={vals.shape[0]} s={vals.shape[1]} T={T} best={score[0] if len(score) else None!r}")
    np.savez_compressed(os.path.join(HERE, f"pipe_{name}.npz"), **arrays)


if __name__ == "__main__":
    main()
