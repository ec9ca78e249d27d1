"""A small workload touching every kernel family once, for compute-sanitizer (racecheck /
synccheck / memcheck): screened n = 2, 3, 4 searches (TMA + mbarrier sweeps, seeds, merge),
the INT8 Ozaki Gram (tcgen05 + TMEM + TMA), the QR screen, the exact kernels, SIS scores and
the final-rung evaluator, the INT8 Gram fix-up rows, the double-double ill-tuple screen and
the tile-screened dim-3 / dim-4 sweeps.
Checks every result against the oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from oracle import oracle as orc  # noqa: E402
from paper_2502_20072_b200 import L0Config, SearchStats, _lib, l0_search  # noqa: E402


def check(got, want):
    assert [g.indices for g in got] == [w["indices"] for w in want], ([g.indices for g in got], [w["indices"] for w in want])
    assert all(np.float64(g.score).view(np.int64) == np.float64(w["score"]).view(np.int64) for g, w in zip(got, want))


def main():
    orc.build()
    rng = np.random.default_rng(11)
    # Ozaki Gram (m >= 256), screened n = 3 with 2 tasks
    m, s = 260, 400
    v = rng.uniform(0.5, 2.0, size=(m, s))
    y = v[3] - 2 * v[100] + 0.5 * v[259] + 0.01 * rng.standard_normal(s)
    sl = [np.arange(0, s, 2), np.arange(1, s, 2)]
    st = SearchStats()
    got = l0_search(v, y, sl, L0Config(dimension=3), stats=st, mode="fast")
    check(got, orc.l0_search(v, y, sl, 3, 10, "fp64", threads=16))
    eta, oz = _lib.engine(0).stage_info()
    assert oz, "the INT8 Gram path was not taken"
    # n = 2 and n = 4 (with a near-copy: the QR screen and the exact refit of ill tuples)
    v2 = rng.uniform(0.5, 2.0, size=(40, 200))
    v2[30] = v2[2] + 1e-9 * rng.standard_normal(200)
    y2 = v2[2] - v2[9] + 0.5 * v2[20] + 0.25 * v2[33] + 0.02 * rng.standard_normal(200)
    for n in (2, 4):
        got = l0_search(v2, y2, None, L0Config(dimension=n), mode="fast")
        check(got, orc.l0_search(v2, y2, None, n, 10, "fp64", threads=16))
    # large keep (global collect mode) and the exact path (n = 1)
    got = l0_search(v2, y2, None, L0Config(dimension=2, n_models_store=150), mode="fast")
    check(got, orc.l0_search(v2, y2, None, 2, 150, "fp64", threads=16))
    got = l0_search(v2, y2, None, L0Config(dimension=1), mode="exact")
    check(got, orc.l0_search(v2, y2, None, 1, 10, "fp64", threads=16))
    # spiky rows and a spiky property: INT8 Gram with fp64 fix-up rows (k_oz_fixup)
    vs = v.copy()
    for f in (7, 77, 177):
        vs[f, rng.integers(s)] += 40.0
    ys = y.copy()
    ys[rng.integers(s)] += 3.0
    got = l0_search(vs, ys, sl, L0Config(dimension=3), mode="fast")
    check(got, orc.l0_search(vs, ys, sl, 3, 10, "fp64", threads=16))
    assert _lib.engine(0).stage_loose_rows() > 0, "no loose rows"
    # ill tuples through the double-double Gram screen (ddgram.cu)
    os.environ["L0S_QR_SCREEN"] = "dd"
    got = l0_search(v2, y2, None, L0Config(dimension=4), mode="fast")
    check(got, orc.l0_search(v2, y2, None, 4, 10, "fp64", threads=16))
    del os.environ["L0S_QR_SCREEN"]
    # the tile-screened sweeps (k_tile_max + k_fit3<.., true>, fit4's screened kernel) on planted
    # properties, one task (the screen engages: n_screen counts the tile tests)
    for n, m3, seed in ((3, 200, 31), (4, 100, 32)):
        r3 = np.random.default_rng(seed)
        v3 = r3.uniform(0.5, 2.0, size=(m3, 1000))
        y3 = 2.0 * v3[3] - v3[m3 // 2] + 0.5 * v3[m3 - 9] + (0.3 * v3[m3 // 3] if n == 4 else 0.0) \
            + 0.01 * r3.standard_normal(1000)
        st3 = SearchStats()
        got = l0_search(v3, y3, None, L0Config(dimension=n), stats=st3, mode="fast")
        check(got, orc.l0_search(v3, y3, None, n, 10, "fp64", threads=16))
        print(f"tile screen n={n}: n_screen {st3.device.get('n_screen')}", flush=True)
    # SIS scores
    eng = _lib.engine(0)
    eng.sis_prepare(np.stack([y, y ** 2]), np.concatenate(sl), np.array([0, 200, 400]))
    sc = eng.sis_scores(v[:64])
    assert np.all(np.isfinite(sc))
    print("sanitize probe ok")


if __name__ == "__main__":
    main()
