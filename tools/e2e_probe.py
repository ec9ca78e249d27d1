"""Break down one end-to-end l0_search call on C3 (host-side phases) -- run under gpurun."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_20072_b200 import L0Config, SearchStats, _lib, l0_search  # noqa: E402
from paper_2502_20072_b200.search import _partition  # noqa: E402


def main():
    v, y, slices = bench.make_c3()
    vh = torch.from_numpy(v).pin_memory().numpy()
    yh = torch.from_numpy(y).pin_memory().numpy()
    cfg = L0Config(dimension=3)
    for _ in range(3):
        l0_search(vh, yh, slices, cfg)
    torch.cuda.synchronize()
    for it in range(3):
        st = SearchStats()
        t0 = time.perf_counter()
        l0_search(vh, yh, slices, cfg, stats=st)
        t1 = time.perf_counter()
        d = st.device
        print(f"l0_search pinned: {1e3 * (t1 - t0):.2f} ms  device total {d['ms_total']:.2f} fit {d['ms_fit']:.2f} "
              f"exact {d['ms_exact']:.2f} launches {d['n_launches']} fit_launches {d['n_fit_launches']} "
              f"cands {d['n_candidates']} ill {d['n_ill']} certified {d['certified']} rescans {d['n_rescan']}")
    for it in range(2):
        t0 = time.perf_counter()
        l0_search(v, y, slices, cfg)
        print(f"l0_search pageable: {1e3 * (time.perf_counter() - t0):.2f} ms")
    eng = _lib.engine(0)
    perm, bounds, _ = _partition(v.shape[1], slices)
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.stage(vh, yh, perm, bounds, "fp64")
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        sc, rk, coef, ssr, st = eng.search(3, 10, 0, 2**63 - 1, "fast")
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"stage {1e3 * (t1 - t0):.2f} ms  search {1e3 * (t2 - t1):.2f} ms  (dev gram {st.ms_gram:.2f} "
              f"total {st.ms_total:.2f} fit {st.ms_fit:.2f} exact {st.ms_exact:.2f})")
    x = torch.empty(v.size, dtype=torch.float64, device="cuda")
    src = torch.from_numpy(vh.reshape(-1))
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"raw H2D {v.nbytes / 1e6:.0f} MB: {1e3 * dt:.2f} ms ({v.nbytes / dt / 1e9:.1f} GB/s)")
    # what pinning the caller's pageable pages in place would cost (cudaHostRegister)
    import ctypes

    cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
    if cudart is not None:
        for it in range(3):
            w = np.array(v)
            t0 = time.perf_counter()
            rc = cudart.cudaHostRegister(ctypes.c_void_p(w.ctypes.data), ctypes.c_size_t(w.nbytes), 0)
            t1 = time.perf_counter()
            cudart.cudaHostUnregister(ctypes.c_void_p(w.ctypes.data))
            t2 = time.perf_counter()
            print(f"cudaHostRegister 160 MB rc={rc}: {1e3 * (t1 - t0):.2f} ms, unregister {1e3 * (t2 - t1):.2f} ms")
    for it in range(4):
        t0 = time.perf_counter()
        l0_search(v, y, slices, cfg)
        print(f"l0_search pageable: {1e3 * (time.perf_counter() - t0):.2f} ms")


if __name__ == "__main__":
    main()
