// fsbm_group.cuh -- multi-GPU coalescence step; included by fsbm_coal.cu.
//
// Microphysics is column-local: coal_step touches only its own point, so a
// domain shards into independent i-slabs or WRF-style j-patches (decompose,
// proj/src/driver.cpp:187-196) with no halo and no data-path exchange.  A group owns one
// fsbm_ctx per local device and steps every local shard from its own host thread (the
// reference runs one std::thread per chunk, driver.cpp:56-84).  What crosses shards is the
// end-of-step bookkeeping only:
//   * counters (triples, points, kernel_evals)                      -> sum
//   * the status, by error precedence                               -> max
//   * the first failing point in serial (tile, j, k, i) order        -> min key, then the
//     winner's (category, bin, value, i, k, j)                        -> sum (one contributor)
//   * optional diagnostics: number and mass per category before/after -> sum, kernel ms -> max
// Shards of this process are combined on the host; across processes (one group per
// process, e.g. one rank per GPU under torchrun) the same combine is one NCCL all-reduce
// group of ~250 bytes over NVLink, issued here in C++.  NCCL is dlopen'ed
// (libnccl.so.2) so single-process use never needs it.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <thread>

namespace {

struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

int nccl_api(NcclApi **out) {
    static NcclApi api;
    static std::once_flag once;
    static std::string why;
    std::call_once(once, [] {
        // the process's NCCL if one is loaded already (torch's), else the system's
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            why = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
            return;
        }
        api.h = h;
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllReduce ||
            !api.GroupStart || !api.GroupEnd || !api.GetErrorString) {
            why = "libnccl.so.2 lacks a required symbol";
            api.h = nullptr;
        }
    });
    if (!api.h) return fail(FSBM_CUDA, "NCCL: " + why);
    *out = &api;
    return FSBM_OK;
}

/// Error precedence when shards disagree: the reference validates the plan and shapes,
/// then the stale mask / arguments, before any point runs; device failures trump all.
int status_rank(int st) {
    switch (st) {
    case FSBM_OK: return 0;
    case FSBM_STIFFNESS: return 1;
    case FSBM_DOMAIN: return 2;
    case FSBM_SHAPE: return 3;
    case FSBM_CONFIG: return 4;
    case FSBM_ALLOC: return 5;
    case FSBM_CUDA: return 6;
    default: return 7;
    }
}
int status_of_rank(int r) {
    static const int st[8] = {FSBM_OK, FSBM_STIFFNESS, FSBM_DOMAIN, FSBM_SHAPE,
                              FSBM_CONFIG, FSBM_ALLOC, FSBM_CUDA, FSBM_INTERNAL};
    return st[std::min(std::max(r, 0), 7)];
}

/// Serial-order key of a failing point over the whole domain: (tile, j, k, i), tiles in
/// patch-major order (run_chunks per tile, driver.cpp:384-430) -- comparable across shards
/// without knowing the global extents.  ~0 = no failure.
unsigned long long serial_key(const fsbm_error &e, const fsbm_tile *tiles, int ntiles) {
    unsigned long long t = 0;
    for (int q = 0; q < ntiles; ++q)
        if (e.i >= tiles[q].its && e.i <= tiles[q].ite && e.j >= tiles[q].jts && e.j <= tiles[q].jte) {
            t = static_cast<unsigned long long>(q);
            break;
        }
    return (t << 50) | (static_cast<unsigned long long>(e.j) << 32) |
           (static_cast<unsigned long long>(e.k) << 18) | static_cast<unsigned long long>(e.i);
}

/// One shard's (or one process's) step outcome, the unit the combine works on.
struct StepResult {
    unsigned long long cnt[3] = {0, 0, 0};
    unsigned long long key = ~0ull;
    unsigned long long status = 0; // status_rank
    double err[6] = {0, 0, 0, 0, 0, 0}; // category, bin, value, i, k, j of the key's point
    double diag[4 * FSBM_NCAT] = {};
    double kernel_ms = 0.0;
    std::string msg;
};

void combine(StepResult &acc, const StepResult &r) {
    for (int q = 0; q < 3; ++q) acc.cnt[q] += r.cnt[q];
    if (r.key < acc.key) {
        acc.key = r.key;
        std::copy(r.err, r.err + 6, acc.err);
    }
    if (r.status > acc.status || (r.status == acc.status && acc.msg.empty())) {
        acc.status = r.status;
        acc.msg = r.msg;
    }
    for (int q = 0; q < 4 * FSBM_NCAT; ++q) acc.diag[q] += r.diag[q];
    acc.kernel_ms = std::max(acc.kernel_ms, r.kernel_ms);
}

} // namespace

struct fsbm_group {
    std::vector<int> devices;
    std::vector<fsbm_ctx *> ctx;
    int rank = 0, nranks = 1;
    NcclApi *nccl = nullptr;
    ncclComm_t comm = nullptr;
    cudaStream_t comm_stream = nullptr;
    double *d_buf = nullptr; // device staging of the all-reduce payload
    float last_ms = 0.0f;
};

namespace {

/// The device-path combine across processes: one NCCL group (sum / min / max), then the
/// winner's error payload if the global status is a stiffness failure.
int allreduce_result(fsbm_group *g, StepResult &r) {
    if (g->nranks == 1) return FSBM_OK;
    DeviceGuard dg(g->devices[0]);
    constexpr int kU = 5, kF = 4 * FSBM_NCAT + 1;
    unsigned long long hu[kU] = {r.cnt[0], r.cnt[1], r.cnt[2], r.key, r.status};
    double hf[kF];
    std::copy(r.diag, r.diag + 4 * FSBM_NCAT, hf);
    hf[4 * FSBM_NCAT] = r.kernel_ms;
    auto *du = reinterpret_cast<unsigned long long *>(g->d_buf);
    double *df = g->d_buf + kU, *de = df + kF;
    cudaStream_t s = g->comm_stream;
    FSBM_CUDA_TRY(cudaMemcpyAsync(du, hu, sizeof hu, cudaMemcpyHostToDevice, s));
    FSBM_CUDA_TRY(cudaMemcpyAsync(df, hf, sizeof hf, cudaMemcpyHostToDevice, s));
    NcclApi &N = *g->nccl;
    auto nck = [&](ncclResult_t e) { return e == ncclSuccess ? FSBM_OK : fail(FSBM_CUDA, std::string("NCCL all-reduce: ") + N.GetErrorString(e)); };
    if (int st = nck(N.GroupStart())) return st;
    N.AllReduce(du, du, 3, ncclUint64, ncclSum, g->comm, s);
    N.AllReduce(du + 3, du + 3, 1, ncclUint64, ncclMin, g->comm, s);
    N.AllReduce(du + 4, du + 4, 1, ncclUint64, ncclMax, g->comm, s);
    N.AllReduce(df, df, 4 * FSBM_NCAT, ncclFloat64, ncclSum, g->comm, s);
    N.AllReduce(df + 4 * FSBM_NCAT, df + 4 * FSBM_NCAT, 1, ncclFloat64, ncclMax, g->comm, s);
    if (int st = nck(N.GroupEnd())) return st;
    FSBM_CUDA_TRY(cudaMemcpyAsync(hu, du, sizeof hu, cudaMemcpyDeviceToHost, s));
    FSBM_CUDA_TRY(cudaMemcpyAsync(hf, df, sizeof hf, cudaMemcpyDeviceToHost, s));
    FSBM_CUDA_TRY(cudaStreamSynchronize(s));
    const unsigned long long local_key = r.key;
    std::copy(hu, hu + 3, r.cnt);
    r.key = hu[3];
    if (hu[4] != r.status) r.msg.clear(); // another rank failed first / worse
    r.status = hu[4];
    std::copy(hf, hf + 4 * FSBM_NCAT, r.diag);
    r.kernel_ms = hf[4 * FSBM_NCAT];
    if (r.key != ~0ull) { // the winner's (category, bin, value, i, k, j): one contributor
        double he[6] = {0, 0, 0, 0, 0, 0};
        if (local_key == r.key) std::copy(r.err, r.err + 6, he);
        FSBM_CUDA_TRY(cudaMemcpyAsync(de, he, sizeof he, cudaMemcpyHostToDevice, s));
        if (int st = nck(N.AllReduce(de, de, 6, ncclFloat64, ncclSum, g->comm, s))) return st;
        FSBM_CUDA_TRY(cudaMemcpyAsync(he, de, sizeof he, cudaMemcpyDeviceToHost, s));
        FSBM_CUDA_TRY(cudaStreamSynchronize(s));
        std::copy(he, he + 6, r.err);
    }
    return FSBM_OK;
}

/// Publish a combined result through the single-device outputs / fsbm_last_error.
int finish(fsbm_group *g, StepResult &r, fsbm_counters *counters_out, fsbm_error *err_out,
           fsbm_diag *diag_out) {
    g->last_ms = static_cast<float>(r.kernel_ms);
    if (counters_out) *counters_out = fsbm_counters{r.cnt[0], r.cnt[1], r.cnt[2]};
    if (err_out) *err_out = fsbm_error{-1, -1, 0, 0, 0, 0, 0.0};
    if (diag_out) {
        for (int q = 0; q < FSBM_NCAT; ++q) {
            diag_out->number_before[q] = r.diag[q];
            diag_out->mass_before[q] = r.diag[FSBM_NCAT + q];
            diag_out->number_after[q] = r.diag[2 * FSBM_NCAT + q];
            diag_out->mass_after[q] = r.diag[3 * FSBM_NCAT + q];
        }
        diag_out->coal_kernel_ms_max = static_cast<float>(r.kernel_ms);
    }
    const int st = status_of_rank(static_cast<int>(r.status));
    if (st == FSBM_OK) return FSBM_OK;
    if (st == FSBM_STIFFNESS) {
        const int cat = static_cast<int>(r.err[0]), bin = static_cast<int>(r.err[1]);
        const int i = static_cast<int>(r.err[3]), k = static_cast<int>(r.err[4]),
                  j = static_cast<int>(r.err[5]);
        if (err_out) *err_out = fsbm_error{cat, bin, 1, i, k, j, r.err[2]};
        return fail(FSBM_STIFFNESS, stiffness_message(cat, bin, r.err[2]) + " at grid point (i=" +
                                        std::to_string(i) + ", k=" + std::to_string(k) +
                                        ", j=" + std::to_string(j) + ")");
    }
    return fail(st, r.msg.empty() ? "fissioned_step: a shard on another rank failed (status " +
                                        std::to_string(st) + ")"
                                  : r.msg);
}

/// Run fn(d) for every local device, each from its own host thread.
template <typename F> void for_each_device(fsbm_group *g, F &&fn) {
    const int n = static_cast<int>(g->ctx.size());
    if (n == 1) {
        fn(0);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(n);
    for (int d = 0; d < n; ++d) th.emplace_back([&fn, d] { fn(d); });
    for (auto &t : th) t.join();
}

StepResult shard_result(int st, const fsbm_counters &cnt, const fsbm_error &e,
                        const fsbm_tile *tiles, int ntiles, fsbm_ctx *c) {
    StepResult r;
    r.cnt[0] = cnt.triples;
    r.cnt[1] = cnt.points;
    r.cnt[2] = cnt.kernel_evals;
    r.status = status_rank(st);
    if (st != FSBM_OK) r.msg = fsbm_last_error();
    if (st == FSBM_STIFFNESS && e.has_point) {
        r.key = serial_key(e, tiles, ntiles);
        r.err[0] = e.category;
        r.err[1] = e.bin;
        r.err[2] = e.value;
        r.err[3] = e.i;
        r.err[4] = e.k;
        r.err[5] = e.j;
    }
    float ms = 0.0f;
    if (st == FSBM_OK || st == FSBM_STIFFNESS) fsbm_ctx_last_timing(c, &ms, nullptr);
    r.kernel_ms = ms;
    return r;
}

} // namespace

extern "C" {

int fsbm_decompose(fsbm_ranges global, int nshards, int split, fsbm_ranges *out) {
    if (!out) return fail(FSBM_DOMAIN, "decompose: null output");
    if (split != FSBM_SPLIT_I && split != FSBM_SPLIT_J)
        return fail(FSBM_CONFIG, "decompose: split must be FSBM_SPLIT_I or FSBM_SPLIT_J");
    const int lo = split == FSBM_SPLIT_I ? global.ids : global.jds;
    const int hi = split == FSBM_SPLIT_I ? global.ide : global.jde;
    const int extent = hi - lo + 1;
    if (nshards < 1 || nshards > extent) // split_range (driver.cpp:35-51)
        return fail(FSBM_DOMAIN, std::string("decompose: ") + (split == FSBM_SPLIT_I ? "i-slab" : "patch") +
                                     " count " + std::to_string(nshards) + " does not fit extent " +
                                     std::to_string(extent));
    const int base = extent / nshards, rem = extent % nshards;
    int start = lo;
    for (int p = 0; p < nshards; ++p) {
        const int len = base + (p < rem ? 1 : 0);
        out[p] = global;
        if (split == FSBM_SPLIT_I) {
            out[p].ids = start;
            out[p].ide = start + len - 1;
        } else {
            out[p].jds = start;
            out[p].jde = start + len - 1;
        }
        start += len;
    }
    return FSBM_OK;
}

int fsbm_nccl_unique_id(uint8_t id[128]) {
    if (!id) return fail(FSBM_DOMAIN, "nccl id: null output");
    NcclApi *N = nullptr;
    if (int st = nccl_api(&N)) return st;
    ncclUniqueId u;
    if (ncclResult_t e = N->GetUniqueId(&u); e != ncclSuccess)
        return fail(FSBM_CUDA, std::string("ncclGetUniqueId: ") + N->GetErrorString(e));
    static_assert(sizeof(u) == 128, "ncclUniqueId size");
    std::memcpy(id, &u, 128);
    return FSBM_OK;
}

int fsbm_group_create(int ndev, const int *devices, int rank, int nranks, const uint8_t *nccl_id,
                      int nkr, const double *x, double ratio, int npairs, const int *pair_abd,
                      const double *t750, const double *t500, fsbm_group **out) {
    if (!out) return fail(FSBM_DOMAIN, "fsbm_group_create: null output");
    *out = nullptr;
    if (ndev < 1 || !devices) return fail(FSBM_DOMAIN, "fsbm_group_create: need >= 1 device");
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return fail(FSBM_DOMAIN, "fsbm_group_create: bad rank / nranks");
    if (nranks > 1 && !nccl_id)
        return fail(FSBM_DOMAIN, "fsbm_group_create: nranks > 1 needs the NCCL unique id of rank 0");
    auto *g = new fsbm_group();
    g->rank = rank;
    g->nranks = nranks;
    g->devices.assign(devices, devices + ndev);
    int st = FSBM_OK;
    for (int d = 0; d < ndev && !st; ++d) {
        fsbm_ctx *c = nullptr;
        st = fsbm_ctx_create(devices[d], nkr, x, ratio, npairs, pair_abd, t750, t500, &c);
        if (!st) g->ctx.push_back(c);
    }
    if (!st && nranks > 1) {
        st = nccl_api(&g->nccl);
        if (!st) {
            DeviceGuard dg(devices[0]);
            ncclUniqueId u;
            std::memcpy(&u, nccl_id, 128);
            if (cudaStreamCreateWithFlags(&g->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
                cudaMalloc(&g->d_buf, 64 * sizeof(double)) != cudaSuccess)
                st = fail(FSBM_CUDA, "fsbm_group_create: allocation failed");
            else if (ncclResult_t e = g->nccl->CommInitRank(&g->comm, nranks, u, rank); e != ncclSuccess)
                st = fail(FSBM_CUDA, std::string("ncclCommInitRank: ") + g->nccl->GetErrorString(e));
        }
    }
    if (st) {
        fsbm_group_destroy(g);
        return st;
    }
    *out = g;
    return FSBM_OK;
}

int fsbm_group_destroy(fsbm_group *g) {
    if (!g) return FSBM_OK;
    if (g->comm) g->nccl->CommDestroy(g->comm);
    if (!g->devices.empty()) {
        DeviceGuard dg(g->devices[0]);
        if (g->d_buf) cudaFree(g->d_buf);
        if (g->comm_stream) cudaStreamDestroy(g->comm_stream);
    }
    for (fsbm_ctx *c : g->ctx) fsbm_ctx_destroy(c);
    delete g;
    return FSBM_OK;
}

int fsbm_group_ctx(fsbm_group *g, int local, fsbm_ctx **ctx) {
    if (!g || !ctx || local < 0 || local >= static_cast<int>(g->ctx.size()))
        return fail(FSBM_DOMAIN, "fsbm_group_ctx: bad argument");
    *ctx = g->ctx[local];
    return FSBM_OK;
}

int fsbm_group_step_device(fsbm_group *g, const fsbm_shard *shards, double dt, int substeps,
                           const fsbm_plan *plan, const fsbm_tile *tiles, int ntiles,
                           fsbm_counters *counters_out, fsbm_error *err_out, fsbm_diag *diag_out) {
    if (!g || !shards) return fail(FSBM_DOMAIN, "fsbm_group_step_device: null argument");
    const int n = static_cast<int>(g->ctx.size());
    std::vector<StepResult> res(n);
    for_each_device(g, [&](int d) {
        fsbm_ctx *c = g->ctx[d];
        const fsbm_shard &sh = shards[d];
        const size_t np = static_cast<size_t>(sh.ranges.ide - sh.ranges.ids + 1) *
                          (sh.ranges.kde - sh.ranges.kds + 1) * (sh.ranges.jde - sh.ranges.jds + 1);
        double before[2 * FSBM_NCAT] = {}, after[2 * FSBM_NCAT] = {};
        int st = FSBM_OK;
        if (diag_out) st = fsbm_state_moments_device(c, np, sh.bins, before, sh.stream);
        fsbm_counters cnt{0, 0, 0};
        fsbm_error e{-1, -1, 0, 0, 0, 0, 0.0};
        if (!st)
            st = fsbm_step_grid_device(c, sh.ranges, sh.bins, sh.pressure, sh.temperature, sh.mask,
                                       dt, substeps, plan, tiles, ntiles, sh.stream, &cnt, &e);
        StepResult r = shard_result(st, cnt, e, tiles, ntiles, c);
        if (diag_out && st == FSBM_OK) {
            if (int s2 = fsbm_state_moments_device(c, np, sh.bins, after, sh.stream)) {
                r.status = status_rank(s2);
                r.msg = fsbm_last_error();
            }
            std::copy(before, before + 2 * FSBM_NCAT, r.diag);
            std::copy(after, after + 2 * FSBM_NCAT, r.diag + 2 * FSBM_NCAT);
        }
        res[d] = std::move(r);
    });
    StepResult acc;
    for (const StepResult &r : res) combine(acc, r);
    if (int st = allreduce_result(g, acc)) return st;
    return finish(g, acc, counters_out, err_out, diag_out);
}

int fsbm_group_step_host(fsbm_group *g, fsbm_ranges global, int split,
                         double *const bins_h[FSBM_NCAT], const double *pressure_h,
                         const double *temperature_h, const uint8_t *mask_h, double dt,
                         int substeps, const fsbm_plan *plan, const fsbm_tile *tiles, int ntiles,
                         fsbm_counters *counters_out, fsbm_error *err_out) {
    if (!g) return fail(FSBM_DOMAIN, "fsbm_group_step_host: null group");
    const int n = static_cast<int>(g->ctx.size());
    const int total = n * g->nranks;
    std::vector<fsbm_ranges> parts(total);
    if (int st = fsbm_decompose(global, total, split, parts.data())) return st;
    std::vector<StepResult> res(n);
    for_each_device(g, [&](int d) {
        fsbm_ctx *c = g->ctx[d];
        fsbm_counters cnt{0, 0, 0};
        fsbm_error e{-1, -1, 0, 0, 0, 0, 0.0};
        const int st = fsbm_step_patch_host(c, global, parts[g->rank * n + d], bins_h, pressure_h,
                                            temperature_h, mask_h, dt, substeps, plan, tiles,
                                            ntiles, &cnt, &e);
        res[d] = shard_result(st, cnt, e, tiles, ntiles, c);
    });
    StepResult acc;
    for (const StepResult &r : res) combine(acc, r);
    if (int st = allreduce_result(g, acc)) return st;
    return finish(g, acc, counters_out, err_out, nullptr);
}

int fsbm_group_last_timing(const fsbm_group *g, float *coal_kernel_ms_max) {
    if (!g || !coal_kernel_ms_max) return fail(FSBM_DOMAIN, "null argument");
    *coal_kernel_ms_max = g->last_ms;
    return FSBM_OK;
}

} // extern "C"
