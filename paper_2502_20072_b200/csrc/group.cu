// group.cu -- one search over several devices of one process (the drop-in's `workers`).
//
// The reference parallelises l0_search in-process: `workers` threads pull contiguous rank
// ranges and their top lists are merged by (score, rank) (search.py:258-304).  Here a group
// owns one context per device and one host thread per device:
//
//   stage  : device g uploads row block g of the (m, s) inputs from the host (its own PCIe
//            link; pageable sources through the pinned ring, hostcopy.cu), the blocks are
//            exchanged device to device (cudaMemcpyPeerAsync over NVLink / NVSwitch), and
//            every device stages the whole problem from its local copy (l0s_stage, device
//            inputs: gather, normalize, INT8 Gram, flags -- 0.6 ms at C3, cheaper than a Gram
//            shard plus its exchange);
//   search : device g searches part g of G (l0s_search_part: every G-th unit of the screened
//            sweep, else the contiguous rank range), certifying its own top list exactly;
//   merge  : the parts' lists merge by (score, rank) on the host (search.py:303), records
//            (coefficients, per-task ssr) travel with their entries.
//
// Devices may repeat (several contexts on one device): the same code path, used by the tests
// on a one-GPU box.
#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/l0search.h"
#include "kernels.h"

using namespace l0s;

struct l0s_group {
    std::vector<int> dev;
    std::vector<l0s_ctx*> ctx;
    std::vector<double*> xin;  // per member: full (m, s) input copy
    std::vector<double*> yin;
    std::vector<int64_t*> pin;
    std::vector<size_t> cap;   // bytes of xin
    std::vector<HostStager*> stager;
    std::vector<cudaStream_t> st;
    int64_t m = 0, s = 0;
    int T = 0;
    bool staged = false;
};

namespace {

// Run f(g) on one host thread per member; the first failing member's status and message win.
template <typename F>
int run_all(l0s_group* g, F f) {
    const int G = (int)g->ctx.size();
    std::vector<int> rc(G, L0S_OK);
    std::vector<std::string> msg(G);
    std::vector<std::thread> th;
    for (int i = 0; i < G; ++i)
        th.emplace_back([&, i] {
            cudaSetDevice(g->dev[i]);
            rc[i] = f(i);
            if (rc[i]) msg[i] = l0s_last_error();
        });
    for (auto& t : th) t.join();
    for (int i = 0; i < G; ++i)
        if (rc[i]) return set_error(rc[i], ("device member " + std::to_string(i) + ": " + msg[i]).c_str());
    return L0S_OK;
}

// The parts' exchange (l0s_set_part_exchange) inside one process: every member thread brings
// its best exact scores; the last to arrive merges them and wakes the others with the keep-th
// of the union.  A member that fails before arriving aborts the round (the others get +inf
// and certify against their own lists).
struct PartExchange {
    std::mutex mu;
    std::condition_variable cv;
    int G = 0, arrived = 0;
    int64_t keep = 0;
    bool aborted = false;
    std::vector<double> all;
    double result = INFINITY;
    bool done = false;

    static double call(const double* scores, int64_t count, void* user) {
        auto* x = static_cast<PartExchange*>(user);
        std::unique_lock<std::mutex> lk(x->mu);
        x->all.insert(x->all.end(), scores, scores + count);
        if (++x->arrived == x->G) {
            std::sort(x->all.begin(), x->all.end());
            x->result = (int64_t)x->all.size() >= x->keep ? x->all[(size_t)x->keep - 1] : INFINITY;
            x->done = true;
            x->cv.notify_all();
        } else {
            x->cv.wait(lk, [x] { return x->done || x->aborted; });
        }
        return x->done ? x->result : INFINITY;
    }
    void abort() {
        std::lock_guard<std::mutex> lk(mu);
        aborted = true;
        cv.notify_all();
    }
};

int cuda_fail(cudaError_t e, const char* what) {
    return set_error(L0S_ECUDA, (std::string(what) + ": " + cudaGetErrorString(e)).c_str());
}

void release_inputs(l0s_group* g, int i) {
    cudaSetDevice(g->dev[i]);
    if (g->xin[i]) cudaFree(g->xin[i]);
    if (g->yin[i]) cudaFree(g->yin[i]);
    if (g->pin[i]) cudaFree(g->pin[i]);
    g->xin[i] = nullptr;
    g->yin[i] = nullptr;
    g->pin[i] = nullptr;
    g->cap[i] = 0;
}

struct Entry {
    double score;
    int64_t rank;
    int member;
    int64_t index;
};

}  // namespace

extern "C" {

int l0s_group_create(int ndev, const int* devices, l0s_group** out) {
    *out = nullptr;
    if (ndev < 1 || !devices) return set_error(L0S_EINVAL, "need at least one device");
    l0s_group* g = new l0s_group();
    for (int i = 0; i < ndev; ++i) {
        l0s_ctx* c = nullptr;
        const int rc = l0s_create(devices[i], &c);
        if (rc) {
            const std::string msg = l0s_last_error();
            l0s_group_destroy(g);
            return set_error(rc, msg.c_str());
        }
        g->dev.push_back(devices[i]);
        g->ctx.push_back(c);
        g->xin.push_back(nullptr);
        g->yin.push_back(nullptr);
        g->pin.push_back(nullptr);
        g->cap.push_back(0);
        g->stager.push_back(nullptr);
        cudaStream_t s = nullptr;
        cudaSetDevice(devices[i]);
        cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        g->st.push_back(s);
    }
    // peer access between distinct devices (NVLink / NVSwitch); a repeated device needs none
    for (int a = 0; a < ndev; ++a)
        for (int b = 0; b < ndev; ++b) {
            if (devices[a] == devices[b]) continue;
            int ok = 0;
            cudaDeviceCanAccessPeer(&ok, devices[a], devices[b]);
            if (ok) {
                cudaSetDevice(devices[a]);
                const cudaError_t e = cudaDeviceEnablePeerAccess(devices[b], 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            }
        }
    *out = g;
    return L0S_OK;
}

int l0s_group_destroy(l0s_group* g) {
    if (!g) return L0S_OK;
    for (size_t i = 0; i < g->ctx.size(); ++i) {
        release_inputs(g, (int)i);
        if (g->stager[i]) host_stager_destroy(g->stager[i]);
        if (g->st[i]) cudaStreamDestroy(g->st[i]);
        l0s_destroy(g->ctx[i]);
    }
    delete g;
    return L0S_OK;
}

int l0s_group_size(l0s_group* g, int* out) {
    if (!g) return set_error(L0S_EINVAL, "null group");
    *out = (int)g->ctx.size();
    return L0S_OK;
}

int l0s_group_ctx(l0s_group* g, int member, l0s_ctx** out) {
    if (!g || member < 0 || member >= (int)g->ctx.size()) return set_error(L0S_EINVAL, "bad group member");
    *out = g->ctx[(size_t)member];
    return L0S_OK;
}

// values (m, s) contiguous, or rows[m] host pointers to s float64 each (exactly one non-null)
int l0s_group_stage(l0s_group* g, const double* values, const double* const* rows, int64_t m, int64_t s,
                    const double* y, const int64_t* perm, const int64_t* bounds, int ntasks, int precision) {
    if (!g) return set_error(L0S_EINVAL, "null group");
    if (m < 1 || s < 1 || ntasks < 1) return set_error(L0S_EINVAL, "need m >= 1, s >= 1, ntasks >= 1");
    if (!values == !rows) return set_error(L0S_EINVAL, "give either a matrix or row pointers");
    g->staged = false;
    const int G = (int)g->ctx.size();
    const size_t bytes = sizeof(double) * (size_t)m * (size_t)s;
    // 1. every member: a full-size input buffer, y and perm, and its row block from the host
    std::vector<int64_t> r0(G + 1);
    for (int i = 0; i <= G; ++i) r0[i] = m * i / G;
    int rc = run_all(g, [&](int i) -> int {
        if (g->cap[i] < bytes) {
            release_inputs(g, i);
            cudaError_t e = cudaMalloc(&g->xin[i], bytes);
            if (e == cudaSuccess) e = cudaMalloc(&g->yin[i], sizeof(double) * s);
            if (e == cudaSuccess) e = cudaMalloc(&g->pin[i], sizeof(int64_t) * s);
            if (e != cudaSuccess) return cuda_fail(e, "group input buffers");
            g->cap[i] = bytes;
        }
        cudaError_t e = cudaMemcpyAsync(g->yin[i], y, sizeof(double) * s, cudaMemcpyHostToDevice, g->st[i]);
        if (e == cudaSuccess) e = cudaMemcpyAsync(g->pin[i], perm, sizeof(int64_t) * s, cudaMemcpyHostToDevice, g->st[i]);
        if (e != cudaSuccess) return cuda_fail(e, "group y / perm upload");
        const int64_t a = r0[i], b = r0[i + 1];
        if (b > a) {
            const void* probe = rows ? (const void*)rows[a] : (const void*)(values + a * s);
            if (!host_is_pinned(probe)) {
                if (!g->stager[i]) g->stager[i] = host_stager_create();
            }
            auto row = [&](int64_t r) -> const void* { return rows ? rows[a + r] : values + (a + r) * s; };
            if (g->stager[i] && !host_is_pinned(probe)) {
                e = host_stager_copy_rows(g->stager[i], g->xin[i] + a * s, row, b - a, sizeof(double) * s, g->st[i]);
            } else {
                for (int64_t r = a; r < b && e == cudaSuccess; ++r)
                    e = cudaMemcpyAsync(g->xin[i] + r * s, row(r - a), sizeof(double) * s, cudaMemcpyHostToDevice,
                                        g->st[i]);
            }
            if (e != cudaSuccess) return cuda_fail(e, "group row upload");
        }
        e = cudaStreamSynchronize(g->st[i]);
        return e == cudaSuccess ? L0S_OK : cuda_fail(e, "group upload");
    });
    if (rc) return rc;
    // 2. every member pulls the other blocks from their owners (device to device)
    rc = run_all(g, [&](int i) -> int {
        for (int o = 0; o < G; ++o) {
            if (o == i || r0[o + 1] == r0[o]) continue;
            const size_t off = (size_t)r0[o] * s, n = sizeof(double) * (size_t)(r0[o + 1] - r0[o]) * s;
            const cudaError_t e = g->dev[o] == g->dev[i]
                                      ? cudaMemcpyAsync(g->xin[i] + off, g->xin[o] + off, n, cudaMemcpyDeviceToDevice, g->st[i])
                                      : cudaMemcpyPeerAsync(g->xin[i] + off, g->dev[i], g->xin[o] + off, g->dev[o], n, g->st[i]);
            if (e != cudaSuccess) return cuda_fail(e, "group block exchange");
        }
        const cudaError_t e = cudaStreamSynchronize(g->st[i]);
        return e == cudaSuccess ? L0S_OK : cuda_fail(e, "group block exchange");
    });
    if (rc) return rc;
    // 3. every member stages the whole problem from its device copy
    rc = run_all(g, [&](int i) -> int {
        return l0s_stage(g->ctx[i], g->xin[i], m, s, g->yin[i], g->pin[i], bounds, ntasks, precision, 1);
    });
    if (rc) return rc;
    g->m = m;
    g->s = s;
    g->T = ntasks;
    g->staged = true;
    return L0S_OK;
}

int l0s_group_search(l0s_group* g, int n, int64_t keep, int mode, double* out_scores, int64_t* out_ranks,
                     double* out_coef, double* out_ssr, int64_t* out_count, l0s_stats* stats) {
    if (out_count) *out_count = 0;
    if (!g || !g->staged) return set_error(L0S_ESTATE, "l0s_group_stage must be called first");
    if (keep < 1) return set_error(L0S_EINVAL, "keep must be >= 1");
    const int G = (int)g->ctx.size();
    const int p = n + 1, T = g->T;
    std::vector<std::vector<double>> sc(G, std::vector<double>((size_t)keep)), cf(G), ss(G);
    std::vector<std::vector<int64_t>> rk(G, std::vector<int64_t>((size_t)keep));
    std::vector<int64_t> cnt(G, 0);
    std::vector<l0s_stats> st(G);
    for (int i = 0; i < G; ++i) {
        cf[i].resize((size_t)keep * T * p);
        ss[i].resize((size_t)keep * T);
    }
    // the parts certify against the keep-th of their union (one exchange per search)
    PartExchange ex;
    ex.G = G;
    ex.keep = keep;
    for (int i = 0; i < G && G > 1; ++i) l0s_set_part_exchange(g->ctx[i], &PartExchange::call, &ex);
    int rc = run_all(g, [&](int i) -> int {
        const int r = l0s_search_part(g->ctx[i], n, keep, i, G, mode, sc[i].data(), rk[i].data(), cf[i].data(),
                                      ss[i].data(), &cnt[i], &st[i]);
        if (r) ex.abort();
        return r;
    });
    for (int i = 0; i < G && G > 1; ++i) l0s_set_part_exchange(g->ctx[i], nullptr, nullptr);
    if (rc) return rc;
    std::vector<Entry> all;
    for (int i = 0; i < G; ++i)
        for (int64_t x = 0; x < cnt[i]; ++x) all.push_back({sc[i][(size_t)x], rk[i][(size_t)x], i, x});
    std::sort(all.begin(), all.end(), [](const Entry& a, const Entry& b) {
        return a.score < b.score || (a.score == b.score && a.rank < b.rank);
    });
    int64_t k = 0;
    for (size_t x = 0; x < all.size() && k < keep; ++x) {
        if (k > 0 && all[x].rank == out_ranks[k - 1]) continue;  // parts are disjoint; defensive
        const Entry& e = all[x];
        out_scores[k] = e.score;
        out_ranks[k] = e.rank;
        if (out_coef)
            std::memcpy(out_coef + k * T * p, cf[e.member].data() + e.index * T * p, sizeof(double) * T * p);
        if (out_ssr) std::memcpy(out_ssr + k * T, ss[e.member].data() + e.index * T, sizeof(double) * T);
        ++k;
    }
    *out_count = k;
    if (stats) {
        l0s_stats a = st[0];
        int64_t total = 0;
        l0s_count(g->m, n, &total);
        for (int i = 1; i < G; ++i) {
            const l0s_stats& b = st[i];
            a.n_tuples += b.n_tuples;
            a.ms_total = std::max(a.ms_total, b.ms_total);
            a.ms_fit = std::max(a.ms_fit, b.ms_fit);
            a.ms_exact = std::max(a.ms_exact, b.ms_exact);
            a.ms_gram = std::max(a.ms_gram, b.ms_gram);
            a.theta = std::max(a.theta, b.theta);
            a.n_candidates += b.n_candidates;
            a.n_ill += b.n_ill;
            a.n_rescan += b.n_rescan;
            a.n_fit_launches = std::max(a.n_fit_launches, b.n_fit_launches);
            a.n_launches += b.n_launches;
            a.certified = a.certified && b.certified;
            a.margin = std::min(a.margin, b.margin);
            a.ms_qr = std::max(a.ms_qr, b.ms_qr);
            a.n_ill_refit += b.n_ill_refit;
            a.ms_gram_kernel = std::max(a.ms_gram_kernel, b.ms_gram_kernel);
            a.ms_records = std::max(a.ms_records, b.ms_records);
            a.n_eval += b.n_eval;
            a.n_screen += b.n_screen;
        }
        a.n_tuples = total;  // parts of one search (screened parts each report the whole range)
        *stats = a;
    }
    return L0S_OK;
}

}  // extern "C"
