// coal_dmma.cuh -- FSBM_NUMERICS_FAST on the FP64 tensor cores (DMMA.8x8x4), nkr in {32, 33}.
//
// Same reassociated mathematics as coal_fast.cuh, restated as small GEMMs over a
// batch of points so that the FP64 tensor pipe does the multiply-adds.  For a pair
// (a, b -> d), pass X, owner o, stream index s, point q:
//
//   row pass    (X=R): o = i, s = j, stream v = nb, owner scale f = na, loss -> a
//   column pass (X=C): o = j, s = i, stream v = na, owner scale f = nb, loss -> b
//     T(o,s)  = K500 / (K750-K500) at cell (i,j)          (self pairs: K(min,max))
//     Y1[o,q] = sum_s T(o,s) v_q[s]                         loss of bin o
//     Y2[o,q] = sum_s T(o,s) clo(o,s) v_q[s]                gain into bin o
//     Y3[o,q] = sum_s T(o,s) chi(o,s) v_q[s]                gain into bin o+1
//   with Y = Y^500 + w_q Y^d (the pressure weight scales output column q, so it is
//   applied once after the GEMM).  delta[loss][o] -= dt f Y1, delta[d][o] += dt f Y2,
//   delta[d][o+1] += dt f Y3.
//
// "Owner-local" cells are those whose Kovetz-Olund targets (GainTable, incl. the top
// rule) all lie in {o, o+1}; their (clo, chi) live in one combined table G[i][j]
// (row-pass coefficients below the diagonal, column-pass on/above it).  Anything
// else is an "exception" cell, gathered per target from a CSR list (none at 33 bins).
//
// GEMM shape: DMMA C[8 rows o x 8 points] += A[8 x 4 s] B[4 s x 8 points].  For an
// owned far cell clo + chi == 1, so Y3 = YG - Y2 with YG = sum T (clo+chi) v; in the
// K-steps where every cell of the 8-row block is owned-far ("full" steps) YG shares
// the loss DMMAs, so only the diagonal ("mixed") steps need a third product.
//
// Work split: warp (g, b) owns rows [8b, 8b+8) for the 16 points of group g over all
// pairs (4 groups x 4 blocks = 16 warps, 64 points per batch).  Its deltas and the hi-gain
// carry of row 8b+7 into the next block live in TMEM (tcgen05.alloc; one 96-column slot
// per warp in its lane quadrant: deterministic, no atomics), which frees the registers
// for 16 warps x 128 (-DFSBM_DMMA_NO_TMEM: the register/shared-memory variant, 12 warps).
// The 33rd (top) row -- 1/8 of a DMMA tile -- is a scalar FP64 dot product split over
// the group's four warps.  Per-pair tables (T500, Kd: one [S][S] layout read row-wise by
// the row pass and transposed by the column pass, both bank-conflict free at pitch
// S = 36) are triple-buffered in smem by 1-D TMA bulk copies; the last warp to release a
// buffer refills it with the pair three ahead, so warps drift freely across pairs.  The
// 33-bin grid is compiled in (nkr, pitch, tail row as immediates) and the unrolled
// K-loops are specialised per block and pass direction.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <string>
#include <vector>

#include "coal_fast.cuh"
#include "fsbm_common.cuh"

namespace fsbm {

// Deltas live in TMEM (tcgen05.ld/st): the 48 registers they free let the CTA run 4 point
// groups (16 warps x 128 registers) instead of 3 (12 x 168) -- measured 96.0 vs 79.9 M upd/s
// at C2 in round 1 (the register variant is retired).

constexpr int kDmmaRB = 4;   // full 8-row blocks handled by this kernel (nkr = 32 or 33)
constexpr int kDmmaNBUF = 2; // per-pair table buffers in flight per half (TMA lookahead)

struct DmmaTables {
    int nkr = 0, S = 0, npairs = 0;
    double *blob = nullptr;  // [pair][T500 | Kd], each [S][S] (row-pass layout), zero padded
    double *gains = nullptr; // [Glo | Ghi], each [S][S], combined owner-local coefficients
    int *exc_off = nullptr;  // [3][nkr+1]  (0 row/cross, 1 row/self, 2 column)
    ExcEntry *exc = nullptr;
    int nexc = 0;
    int kf[3][kDmmaRB] = {}, km[3][kDmmaRB] = {}; // [R-cross, R-self, C][block]
};

inline void free_dmma_tables(DmmaTables &t) {
    cudaFree(t.blob);
    cudaFree(t.gains);
    cudaFree(t.exc_off);
    cudaFree(t.exc);
    t = DmmaTables{};
}

inline int build_dmma_tables(DmmaTables &D, int nkr, int npairs, const std::vector<int> &abd,
                             const double *t750, const double *t500,
                             const std::vector<int32_t> &g_lo, const std::vector<double> &g_wlo,
                             const std::vector<double> &g_whi, const std::vector<double> &g_top) {
    if (nkr / 8 != kDmmaRB || nkr % 8 > 1) return 0; // this kernel is unused for other grids
    const int S = (nkr + 3) / 4 * 4;
    const size_t nn = static_cast<size_t>(S) * S;
    const size_t sq = static_cast<size_t>(nkr) * nkr;
    std::vector<double> blob(static_cast<size_t>(npairs) * 2 * nn, 0.0), G(2 * nn, 0.0);
    for (int p = 0; p < npairs; ++p) {
        const bool self = abd[3 * p] == abd[3 * p + 1];
        const double *k750 = t750 + p * sq, *k500 = t500 + p * sq;
        double *b = blob.data() + static_cast<size_t>(p) * 2 * nn;
        for (int i = 0; i < nkr; ++i)
            for (int j = 0; j < nkr; ++j) {
                const size_t u = self ? static_cast<size_t>(std::min(i, j)) * nkr + std::max(i, j)
                                      : static_cast<size_t>(i) * nkr + j;
                b[static_cast<size_t>(i) * S + j] = k500[u];
                b[nn + static_cast<size_t>(i) * S + j] = k750[u] - k500[u];
            }
    }
    // owner-local coefficients of cell (i,j) for owner o: targets must lie in {o, o+1}
    auto local = [&](int i, int j, int o, double &clo, double &chi) {
        const size_t e = static_cast<size_t>(i) * nkr + j;
        clo = chi = 0.0;
        auto put = [&](int t, double c) {
            if (c == 0.0) return true;
            if (t == o) { clo += c; return true; }
            if (t == o + 1) { chi += c; return true; }
            return false;
        };
        if (g_lo[e] >= 0) return put(g_lo[e], g_wlo[e]) && put(g_lo[e] + 1, g_whi[e]);
        return put(nkr - 1, g_top[e]);
    };
    std::vector<std::vector<ExcEntry>> ex[3];
    for (auto &v : ex) v.assign(nkr, {});
    auto add_exc = [&](int kind, int i, int j, double scale) {
        const size_t e = static_cast<size_t>(i) * nkr + j;
        const int ii = kind == 1 ? std::min(i, j) : i, jj = kind == 1 ? std::max(i, j) : j;
        if (g_lo[e] >= 0) {
            if (g_wlo[e] != 0.0) ex[kind][g_lo[e]].push_back({ii, jj, scale * g_wlo[e]});
            if (g_whi[e] != 0.0) ex[kind][g_lo[e] + 1].push_back({ii, jj, scale * g_whi[e]});
        } else {
            ex[kind][nkr - 1].push_back({ii, jj, scale * g_top[e]});
        }
    };
    for (int i = 0; i < nkr; ++i)
        for (int j = 0; j < nkr; ++j) {
            double clo, chi;
            if (j < i) { // row pass, owner i
                if (local(i, j, i, clo, chi)) {
                    G[static_cast<size_t>(i) * S + j] = clo;
                    G[nn + static_cast<size_t>(i) * S + j] = chi;
                } else {
                    add_exc(0, i, j, 1.0);
                    add_exc(1, i, j, 1.0);
                }
            } else { // column pass, owner j (incl. the diagonal)
                if (local(i, j, j, clo, chi)) {
                    G[static_cast<size_t>(i) * S + j] = clo;
                    G[nn + static_cast<size_t>(i) * S + j] = chi;
                } else {
                    add_exc(2, i, j, 1.0);
                    if (i == j) add_exc(1, i, j, 0.5); // self diagonal: rate halved
                }
            }
        }
    std::vector<int> off(3 * (nkr + 1));
    std::vector<ExcEntry> all;
    for (int k = 0; k < 3; ++k) {
        for (int t = 0; t < nkr; ++t) {
            off[k * (nkr + 1) + t] = static_cast<int>(all.size());
            all.insert(all.end(), ex[k][t].begin(), ex[k][t].end());
        }
        off[k * (nkr + 1) + nkr] = static_cast<int>(all.size());
    }
    D.nexc = static_cast<int>(all.size());
    if (all.empty()) all.push_back({0, 0, 0.0});
    // K-step classes per (pass view, block): 0 every cell owned-far (clo+chi == 1),
    // 2 no owned cell, 1 mixed.  Views: R-cross (s<o), R-self (s<o, s==o at 1/2), C (s<=o).
    auto view = [&](int V, int o, int s, double &lo, double &hi) {
        lo = hi = 0.0;
        if (o >= nkr || s >= nkr) return;
        if (V <= 1) {
            if (s < o) { lo = G[static_cast<size_t>(o) * S + s]; hi = G[nn + static_cast<size_t>(o) * S + s]; }
            else if (V == 1 && s == o) { lo = 0.5 * G[static_cast<size_t>(o) * S + o]; hi = 0.5 * G[nn + static_cast<size_t>(o) * S + o]; }
        } else if (s <= o) {
            lo = G[static_cast<size_t>(s) * S + o];
            hi = G[nn + static_cast<size_t>(s) * S + o];
        }
    };
    const int KS = S / 4;
    for (int V = 0; V < 3; ++V)
        for (int b = 0; b < kDmmaRB; ++b) {
            auto cls = [&](int ks) {
                bool one = true, zero = true;
                for (int r = 0; r < 8; ++r)
                    for (int c = 0; c < 4; ++c) {
                        double lo, hi;
                        view(V, 8 * b + r, 4 * ks + c, lo, hi);
                        one = one && std::fabs(lo + hi - 1.0) <= 4e-16;
                        zero = zero && lo == 0.0 && hi == 0.0;
                    }
                return one ? 0 : zero ? 2 : 1;
            };
            int kf = 0;
            while (kf < KS && cls(kf) == 0) ++kf;
            int km = KS;
            while (km > kf && cls(km - 1) == 2) --km;
            D.kf[V][b] = kf;
            D.km[V][b] = km;
        }
    D.nkr = nkr;
    D.S = S;
    D.npairs = npairs;
    auto up = [](auto **dst, const auto &v) {
        using T = typename std::remove_reference<decltype(v)>::type::value_type;
        return cudaMalloc(reinterpret_cast<void **>(dst), sizeof(T) * v.size()) == cudaSuccess &&
               cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice) == cudaSuccess;
    };
    if (!up(&D.blob, blob) || !up(&D.gains, G) || !up(&D.exc_off, off) || !up(&D.exc, all)) {
        fast_err() = "dmma tables: device allocation failed";
        return 6;
    }
    return 0;
}

// ---- PTX helpers -------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred P1;\n"
                 "WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
                 "r"(parity)
                 : "memory");
}
/// 1-D TMA bulk copy global -> shared, completing on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                             uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
/// 8-byte asynchronous global -> shared copy (LDGSTS: no register round trip).
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
/// D(8x8) += A(8x4) B(4x8), FP64 tensor core.
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// ---- TMEM as the delta store (tcgen05.ld/st, 32x32b shape: thread i <-> TMEM lane base+i) ----
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
/// tcgen05.ld without the wait: the registers are valid only after tm_wait_ld().
__device__ __forceinline__ void tm_ld4_nowait(uint32_t taddr, double (&v)[4]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __hiloint2double(static_cast<int>(r[2 * i + 1]), static_cast<int>(r[2 * i]));
}
__device__ __forceinline__ void tm_st4_nowait(uint32_t taddr, const double (&v)[4]) {
    uint32_t r[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        r[2 * i] = static_cast<uint32_t>(__double2loint(v[i]));
        r[2 * i + 1] = static_cast<uint32_t>(__double2hiint(v[i]));
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }


#ifdef FSBM_DMMA_PROF // per-warp phase cycle counters (A/B profiling builds only)
#define PROF_DECL                                                                                  \
    unsigned long long pf[8] = {};                                                                 \
    unsigned long long pt0 = clock64();
#define PROF_MARK(k)                                                                               \
    {                                                                                              \
        const unsigned long long t1_ = clock64();                                                  \
        pf[k] += t1_ - pt0;                                                                        \
        pt0 = t1_;                                                                                 \
    }
#define PROF_FLUSH                                                                                 \
    if (lane == 0 && F.prof)                                                                       \
        for (int k = 0; k < 8; ++k) atomicAdd(F.prof + wid * 8 + k, pf[k]);
#else
#define PROF_DECL
#define PROF_MARK(k)
#define PROF_FLUSH
#endif
// phases: 0 batch setup, 1 tail, 2 table wait, 3 K-loops, 4 apply barrier, 5 apply..writeback,
// 6 emission, 7 per-pair bookkeeping

struct DmmaArgs {
    unsigned long long *prof; // FSBM_DMMA_PROF builds: [warp][8] cycles per phase
    int S, tail, QP;
    int std_classes; // kf == 2b, km == 2b + 2 in every view and S == 36: unrolled K-loops
    uint32_t nbatches;
    int kf[3][kDmmaRB], km[3][kDmmaRB];
    const double *blob, *gains;
    const int *exc_off;
    const ExcEntry *exc;
    int nexc;
};

constexpr int kDmmaNT = 2;                          // 8-point N-tiles per warp
constexpr int kDmmaG = 4;                           // point groups per CTA (16 points each)
constexpr int kDmmaH = 2;                           // independent halves per CTA
constexpr int kDmmaGH = kDmmaG / kDmmaH;            // point groups per half
constexpr int kDmmaNP = kDmmaG * kDmmaNT * 8;       // 64 points in the CTA's work buffer
constexpr int kDmmaNPH = kDmmaNP / kDmmaH;          // 32 points per half-batch
constexpr int kDmmaThreads = kDmmaG * kDmmaRB * 32; // 512
constexpr int kDmmaHT = kDmmaThreads / kDmmaH;      // 256 threads (8 warps) per half
constexpr int kDmmaQP = (kDmmaNP + 15) / 16 * 16 + 4; // point pitch, = 4 mod 16: conflict-free B fragments

/// register delta add with a runtime (warp-uniform) category
__device__ __forceinline__ void dadd_cat(double (&D)[kNCat][kDmmaNT][2], int cat, int nt, int e,
                                         double v) {
    switch (cat) {
    case 0: D[0][nt][e] += v; break;
    case 1: D[1][nt][e] += v; break;
    case 2: D[2][nt][e] += v; break;
    case 3: D[3][nt][e] += v; break;
    case 4: D[4][nt][e] += v; break;
    default: D[5][nt][e] += v; break;
    }
}

/// One single-half pass of a warp's 8-row block with compile-time K-step classes
/// (full: ks < KF, diagonal: KF <= ks < KM, no owned gains: ks >= KM; KSN steps),
/// fully unrolled so the A-fragment loads/interpolation are scheduled ahead of the
/// DMMA chains.  INTERP: A = K500 + wu*Kd, else A = K500.
template <int KF, int KM, int KSN, bool INTERP, int ASTRIDE>
__device__ __forceinline__ void dmma_pass_single(const double *__restrict__ T5, const double *__restrict__ Td,
                                                 double wu, const double *__restrict__ Glo,
                                                 const double *__restrict__ Ghi, int abase, int /*astride*/,
                                                 const double *__restrict__ vb, int QP, int V, int o, int lc,
                                                 double (&c1)[kDmmaNT][2], double (&c2)[kDmmaNT][2],
                                                 double (&cg)[kDmmaNT][2]) {
    double cf[kDmmaNT][2];
#pragma unroll
    for (int nt = 0; nt < kDmmaNT; ++nt) cf[nt][0] = cf[nt][1] = c2[nt][0] = c2[nt][1] = cg[nt][0] = cg[nt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KSN; ++ks) {
        const int ai = abase + ks * ASTRIDE; // compile-time stride: immediate table offsets
        const double t = INTERP ? fma(wu, Td[ai], T5[ai]) : T5[ai];
        if (ks < KF) { // every cell owned-far: Y3 = YG - Y2 shares the loss DMMAs
            const double t2 = t * Glo[ai];
#pragma unroll
            for (int nt = 0; nt < kDmmaNT; ++nt) {
                const double v = vb[(4 * ks) * QP + nt * 8];
                dmma(cf[nt][0], cf[nt][1], t, v);
                dmma(c2[nt][0], c2[nt][1], t2, v);
            }
        } else if (ks < KM) { // diagonal steps
            const int s = 4 * ks + lc;
            const double msk = V == 2 ? (s <= o ? 1.0 : 0.0) : (s < o ? 1.0 : (V == 1 && s == o ? 0.5 : 0.0));
            const double lo = msk * Glo[ai], hi = msk * Ghi[ai];
            const double t2 = t * lo, tg = t * (lo + hi);
#pragma unroll
            for (int nt = 0; nt < kDmmaNT; ++nt) {
                const double v = vb[(4 * ks) * QP + nt * 8];
                dmma(c1[nt][0], c1[nt][1], t, v);
                dmma(c2[nt][0], c2[nt][1], t2, v);
                dmma(cg[nt][0], cg[nt][1], tg, v);
            }
        } else { // no owned gains
#pragma unroll
            for (int nt = 0; nt < kDmmaNT; ++nt) {
                const double v = vb[(4 * ks) * QP + nt * 8];
                dmma(c1[nt][0], c1[nt][1], t, v);
            }
        }
    }
#pragma unroll
    for (int nt = 0; nt < kDmmaNT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            c1[nt][e] += cf[nt][e];
            cg[nt][e] += cf[nt][e];
        }
}

/// The same pass for a group that straddles a pressure level: A = K500 + w_q Kd with a
/// per-point weight, run as K500 . v + Kd . (w_q v) -- two DMMAs into the same
/// accumulator, the lane's B column scaled by its point's weight wq[nt].
template <int KF, int KM, int KSN, int ASTRIDE>
__device__ __forceinline__ void dmma_pass_dual(const double *__restrict__ T5, const double *__restrict__ Td,
                                               const double (&wq)[kDmmaNT], const double *__restrict__ Glo,
                                               const double *__restrict__ Ghi, int abase,
                                               const double *__restrict__ vb, int QP, int V, int o, int lc,
                                               double (&c1)[kDmmaNT][2], double (&c2)[kDmmaNT][2],
                                               double (&cg)[kDmmaNT][2]) {
    double cf[kDmmaNT][2];
#pragma unroll
    for (int nt = 0; nt < kDmmaNT; ++nt) cf[nt][0] = cf[nt][1] = c2[nt][0] = c2[nt][1] = cg[nt][0] = cg[nt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KSN; ++ks) {
        const int ai = abase + ks * ASTRIDE;
        const double t5 = T5[ai], td = Td[ai];
        double v[kDmmaNT], vw[kDmmaNT];
#pragma unroll
        for (int nt = 0; nt < kDmmaNT; ++nt) {
            v[nt] = vb[(4 * ks) * QP + nt * 8];
            vw[nt] = wq[nt] * v[nt];
        }
        if (ks < KF) {
            const double g = Glo[ai];
#pragma unroll
            for (int nt = 0; nt < kDmmaNT; ++nt) {
                dmma(cf[nt][0], cf[nt][1], t5, v[nt]);
                dmma(cf[nt][0], cf[nt][1], td, vw[nt]);
                dmma(c2[nt][0], c2[nt][1], t5 * g, v[nt]);
                dmma(c2[nt][0], c2[nt][1], td * g, vw[nt]);
            }
        } else if (ks < KM) {
            const int s = 4 * ks + lc;
            const double msk = V == 2 ? (s <= o ? 1.0 : 0.0) : (s < o ? 1.0 : (V == 1 && s == o ? 0.5 : 0.0));
            const double lo = msk * Glo[ai], hi = msk * Ghi[ai];
#pragma unroll
            for (int nt = 0; nt < kDmmaNT; ++nt) {
                dmma(c1[nt][0], c1[nt][1], t5, v[nt]);
                dmma(c1[nt][0], c1[nt][1], td, vw[nt]);
                dmma(c2[nt][0], c2[nt][1], t5 * lo, v[nt]);
                dmma(c2[nt][0], c2[nt][1], td * lo, vw[nt]);
                dmma(cg[nt][0], cg[nt][1], t5 * (lo + hi), v[nt]);
                dmma(cg[nt][0], cg[nt][1], td * (lo + hi), vw[nt]);
            }
        } else {
#pragma unroll
            for (int nt = 0; nt < kDmmaNT; ++nt) {
                dmma(c1[nt][0], c1[nt][1], t5, v[nt]);
                dmma(c1[nt][0], c1[nt][1], td, vw[nt]);
            }
        }
    }
#pragma unroll
    for (int nt = 0; nt < kDmmaNT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            c1[nt][e] += cf[nt][e];
            cg[nt][e] += cf[nt][e];
        }
}

typedef double DmmaAcc[kDmmaNT][2];

/// D[FC] -= L, D[PD] += G with compile-time categories: one indirect branch per pass
/// instead of a branch tree per value.
template <int FC, int PD>
__device__ __forceinline__ void emit_fp(double (&D)[kNCat][kDmmaNT][2], const DmmaAcc &L, const DmmaAcc &G) {
#pragma unroll
    for (int nt = 0; nt < kDmmaNT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            D[FC][nt][e] -= L[nt][e];
            D[PD][nt][e] += G[nt][e];
        }
}

__device__ __forceinline__ void emit_switch(int sel, double (&D)[kNCat][kDmmaNT][2], const DmmaAcc &L,
                                            const DmmaAcc &G) {
#define FSBM_EMIT_CASE(F, P)                                                                       \
    case F * kNCat + P: emit_fp<F, P>(D, L, G); break;
#define FSBM_EMIT_ROW(F)                                                                           \
    FSBM_EMIT_CASE(F, 0) FSBM_EMIT_CASE(F, 1) FSBM_EMIT_CASE(F, 2) FSBM_EMIT_CASE(F, 3)            \
    FSBM_EMIT_CASE(F, 4) FSBM_EMIT_CASE(F, 5)
    switch (sel) {
        FSBM_EMIT_ROW(0)
        FSBM_EMIT_ROW(1)
        FSBM_EMIT_ROW(2)
        FSBM_EMIT_ROW(3)
        FSBM_EMIT_ROW(4)
        FSBM_EMIT_ROW(5)
    default: break;
    }
#undef FSBM_EMIT_ROW
#undef FSBM_EMIT_CASE
}

/// Named barrier over one half of the CTA (ids 1, 2; id 0 is __syncthreads).
__device__ __forceinline__ void half_sync(int h) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + h), "r"(kDmmaHT) : "memory");
}

template <int NKRC>
__global__ void __launch_bounds__(kDmmaThreads, 1) coal_dmma_kernel(StepArgs A, DmmaArgs F) {
    constexpr int NT = kDmmaNT, NP = kDmmaNP, RB = kDmmaRB, NPH = kDmmaNPH, HT = kDmmaHT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // NKRC == 33: the headline grid with its extents compiled in (S = 36, one tail row)
    const int nkr = NKRC ? NKRC : A.nkr, S = NKRC ? (NKRC + 3) / 4 * 4 : F.S, TAIL = NKRC ? NKRC % 8 : F.tail;
    constexpr int QP = kDmmaQP; // compile-time: immediate offsets for the B-fragment loads
    const int KS = S / 4;
    const size_t TBL = static_cast<size_t>(S) * S;
    constexpr int NBUF = kDmmaNBUF;
    // Two independent halves (8 warps, point groups {0,1} and {2,3}) share the CTA's
    // shared memory but nothing else: each steps its own 32-point half-batches with its
    // own table ring and named barrier, so one half's load / apply / stiffness /
    // write-back phases overlap the other half's DMMA K-loops.
    double *tabs = reinterpret_cast<double *>(smem_raw);                 // [H][NBUF][T500|Kd][S][S]
    double *gains = tabs + 2 * kDmmaH * NBUF * TBL;                        // [lo|hi][S][S]
    double *work = gains + 2 * TBL;                                        // [6][S][QP]
    double *tdel = work + static_cast<size_t>(kNCat) * S * QP;             // [6][NP]
    double *wts = tdel + static_cast<size_t>(kNCat) * NP;                  // [NP]
    unsigned long long *act = reinterpret_cast<unsigned long long *>(wts + NP);
    unsigned long long *ptrip = act + NP;
    uint64_t *mbar = reinterpret_cast<uint64_t *>(ptrip + NP);             // [H][NBUF tables], gains
    uint32_t *pidx = reinterpret_cast<uint32_t *>(mbar + kDmmaH * NBUF + 1); // [NP]
    int *pfail = reinterpret_cast<int *>(pidx + NP);                       // [NP]
    __shared__ unsigned long long cta_act[kDmmaH];
    // per point group and category: last bin holding a non-zero value at any live point.
    // Products with an exactly-zero spectrum value vanish (the reference skips rate == 0
    // triples, coalescence.cpp:286-292): a pass whose owner rows are all zero, or whose
    // streamed spectrum is zero, is skipped; the generic (two-half) K-loops also stop at
    // the streamed spectrum's last non-zero bin.  (Cutting K-steps inside the unrolled
    // loops measured slower: the early exits break the schedule.)
    __shared__ int kzg[kDmmaG][kNCat];
    __shared__ int relcnt[kDmmaH][kDmmaNBUF];
    __shared__ short ltop[kNCat * kDmmaNP];
    __shared__ unsigned char nzq[kDmmaNP];
    __shared__ unsigned char wmode_s[kDmmaThreads / 32];

    const int tid = threadIdx.x;
    const int wid = tid >> 5, lane = tid & 31;
    // block b of group g, rotated by g so every SMSP (wid % 4) hosts all four blocks
    // (instruction-cache friendly; the per-block K-loop costs 26/30/34/38 DMMAs balance
    // per SMSP)
    const int g = wid / RB, b = (wid % RB + g) % RB;
    const int h = g / kDmmaGH;                 // this warp's half
    const int htid = tid - h * HT, hwid = htid >> 5, NWH = HT >> 5;
    const int q0 = h * NPH;                    // the half's first point slot
    const int o0 = 8 * b;
    const int lr = lane >> 2, lc = lane & 3;
    const int qg = g * NT * 8;
    const int ot = 8 * RB;                     // the tail (top) row, when TAIL == 1
    if (A.stale && *A.stale) return; // stale mask: the step must not touch the state
    const uint32_t nact = *A.nactive;
    const int npairs = A.pairs.npairs;
    const unsigned long long full_evals = static_cast<unsigned long long>(npairs) * nkr * nkr;
    const int self_tri = nkr * (nkr + 1) / 2, cross_sq = nkr * nkr;
    const double dt = A.dt_sub;
    const uint32_t tbytes = static_cast<uint32_t>(2 * TBL * sizeof(double));
    unsigned long long tr_acc = 0, pt_acc = 0, ev_acc = 0;
    double *htabs = tabs + static_cast<size_t>(h) * NBUF * 2 * TBL;
    uint64_t *hbar = mbar + h * NBUF, *gbar = mbar + kDmmaH * NBUF;

    auto W = [&](int c, int s, int q) -> double & {
        return work[(static_cast<size_t>(c) * S + s) * QP + q];
    };

    if (tid == 0) {
        for (int i = 0; i <= kDmmaH * NBUF; ++i) mbar_init(&mbar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __shared__ uint32_t tmem_base;
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    // this warp's slot: lanes 32*(wid%4).., columns (wid/4)*96: [0,48) deltas, [48,96) carries
    const uint32_t tmw = tmem_base + (static_cast<uint32_t>(32 * (wid & 3)) << 16) + (wid >> 2) * 96;
    if (tid == 0) { // pair-independent gain coefficients, once per CTA
        mbar_expect_tx(gbar, static_cast<uint32_t>(2 * TBL * sizeof(double)));
        tma_bulk_g2s(gains, F.gains, static_cast<uint32_t>(2 * TBL * sizeof(double)), gbar);
    }
    uint32_t pbase = 0; // pairs processed so far by this half: pair #m uses buffer m % NBUF,
                        // phase (m / NBUF) & 1
    bool gains_ready = false;
    // rows [nkr, S) of every category stay zero (K-step padding read by the B fragments)
    for (int f = tid; f < kNCat * (S - nkr) * NP; f += kDmmaThreads) {
        const int q = f % NP, r = f / NP;
        W(r / (S - nkr), nkr + r % (S - nkr), q) = 0.0;
    }
    // the next half-batch's point index and pressure weight (lanes htid < NPH), loaded
    // ahead during the previous half-batch's apply so the batch start does not wait on them
    auto fetch_point = [&](uint32_t hbx, uint32_t &p, double &w) {
        const uint32_t idx = hbx * static_cast<uint32_t>(NPH) + htid;
        const bool live = hbx < F.nbatches && idx < nact;
        p = live ? A.active[idx] : 0xffffffffu; // holes of the level-major list: 0xffffffff
        w = p != 0xffffffffu ? pressure_weight(A.pressure[p]) : 0.0;
    };
    __shared__ uint32_t nx_p[kDmmaNP];
    __shared__ double nx_w[kDmmaNP];
    if (htid < NPH) fetch_point(kDmmaH * blockIdx.x + h, nx_p[q0 + htid], nx_w[q0 + htid]);
    __syncthreads(); // the padding rows are zero for both halves
    PROF_DECL

    for (uint32_t hb = kDmmaH * blockIdx.x + h; hb < F.nbatches && hb * static_cast<uint32_t>(NPH) < nact;
         hb += kDmmaH * gridDim.x) {
        if (htid < NPH) {
            const int q = q0 + htid;
            pidx[q] = nx_p[q];
            wts[q] = nx_w[q];
            pfail[q] = nx_p[q] != 0xffffffffu ? 0 : 1;
            ptrip[q] = 0;
        }
        half_sync(h);
        // spectra -> work by asynchronous copies (LDGSTS), all issued before one wait: a
        // warp instruction covers 4 points x 8 consecutive bins (64-byte runs of each point's
        // spectrum); quads of (category, 4 points) per warp
        constexpr int NQ = kNCat * NPH / 4; // 48 quads per half
        const int qs = lane >> 3, kc = lane & 7;
        for (int u = hwid; u < NQ; u += NWH) {
            const int c = u / (NPH / 4), q = q0 + 4 * (u % (NPH / 4)) + qs;
            const uint32_t p = pidx[q];
            const double *src = A.bins[c] + static_cast<size_t>(p) * nkr;
#pragma unroll
            for (int jj = 0; jj < 5; ++jj) {
                const int k = kc + 8 * jj;
                if (k < nkr) {
                    if (p != 0xffffffffu) cp_async8(&W(c, k, q), src + k);
                    else W(c, k, q) = 0.0;
                }
            }
        }
        cp_async_wait_all();
        // pressure-weight mode of the warp's 16 points, once per half-batch (see the pair loop)
        {
            // holes (padding of a line's last group) take any weight
            const double w0 = wts[qg], wl = wts[qg + (lane & 15)];
            const bool hole = pidx[qg + (lane & 15)] == 0xffffffffu;
            const int wm = __all_sync(0xffffffffu, hole || wl == 0.0)  ? 0
                           : __all_sync(0xffffffffu, hole || wl == w0) ? 1
                                                                       : 2;
            if (lane == 0) wmode_s[wid] = static_cast<unsigned char>(wm);
        }
        half_sync(h);
        for (int u = hwid; u < NQ; u += NWH) { // last non-zero bin per (category, point)
            const int c = u / (NPH / 4), q = q0 + 4 * (u % (NPH / 4)) + qs;
            int top = -1;
#pragma unroll
            for (int jj = 0; jj < 5; ++jj) {
                const int k = kc + 8 * jj;
                if (k < nkr && W(c, k, q) != 0.0) top = k;
            }
#pragma unroll
            for (int d = 1; d < 8; d <<= 1) top = max(top, __shfl_xor_sync(0xffffffffu, top, d));
            if (kc == 0) ltop[c * NP + q] = static_cast<short>(top);
        }
        if (!gains_ready) {
            mbar_wait(gbar, 0);
            gains_ready = true;
        }
        half_sync(h);

        for (int sub = 0; sub < A.substeps; ++sub) {
            if (htid == 0) cta_act[h] = 0ull;
            for (int f = htid; f < kNCat * NPH; f += HT) tdel[(f / NPH) * NP + q0 + f % NPH] = 0.0;
            if (htid < kDmmaGH * kNCat) kzg[h * kDmmaGH + htid / kNCat][htid % kNCat] = -1;
            half_sync(h);
            if (htid < NPH) { // all_zero (coalescence.cpp:270-273)
                const int q = q0 + htid;
                unsigned nz = 0;
                for (int c = 0; c < kNCat; ++c) { // last non-zero bin (the load found it for sub 0)
                    int l = ltop[c * NP + q];
                    if (sub > 0) {
                        l = nkr - 1;
                        while (l >= 0 && W(c, l, q) == 0.0) --l;
                    }
                    nz |= l >= 0 ? (1u << c) : 0u;
                    if (l >= 0 && pfail[q] == 0) atomicMax(&kzg[q / (NT * 8)][c], l);
                }
                unsigned long long m = 0, trip = 0;
                for (int pp = 0; pp < npairs; ++pp)
                    if (nz >> A.pairs.a[pp] & 1u) {
                        m |= 1ull << pp;
                        trip += A.pairs.a[pp] == A.pairs.b[pp] ? self_tri : cross_sq;
                    }
                if (pfail[q] == 0) {
                    act[q] = m;
                    atomicOr(&cta_act[h], m);
                    ptrip[q] += trip;
                } else {
                    act[q] = 0;
                }
                nzq[q] = pfail[q] == 0 ? static_cast<unsigned char>(nz) : 0;
            }
            half_sync(h);
            const unsigned long long amask = cta_act[h];
            // the non-zero-category bits of this lane's four points, 6 bits each: pair p is
            // active at point i iff bit 6i + a[p] is set (coalescence.cpp:270-273)
            uint32_t lnz = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) lnz |= static_cast<uint32_t>(nzq[qg + (i >> 1) * 8 + 2 * lc + (i & 1)]) << (6 * i);

            PROF_MARK(0)
            {
                const double z[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int c = 0; c < 2 * kNCat; ++c) tm_st4_nowait(tmw + 8 * c, z); // deltas, carries
                tm_wait_st();
            }

            // Pair pipeline without barriers (see header), one ring per half.
            auto next_pair = [&](int p) -> int {
                if (p < 0) return -1;
                const unsigned long long rest = amask & ~((2ull << p) - 1ull);
                return rest ? __ffsll(static_cast<long long>(rest)) - 1 : -1;
            };
            int cur = amask ? __ffsll(static_cast<long long>(amask)) - 1 : -1;
            int n = 0;
            if (htid == 0) { // prime all buffers with the first NBUF active pairs
                fence_proxy_async();
                int pp = cur;
                for (int i = 0; i < NBUF; ++i, pp = next_pair(pp)) {
                    const int bi = (pbase + i) % NBUF;
                    relcnt[h][bi] = 0;
                    if (pp >= 0) {
                        mbar_expect_tx(&hbar[bi], tbytes);
                        tma_bulk_g2s(htabs + bi * 2 * TBL, F.blob + static_cast<size_t>(pp) * 2 * TBL, tbytes,
                                     &hbar[bi]);
                    }
                }
            }
            half_sync(h);
            while (cur >= 0) {
                const uint32_t m = pbase + n;
                const int buf = m % NBUF;
                const int nxt = next_pair(cur);
                PROF_MARK(7)
                mbar_wait(&hbar[buf], (m / NBUF) & 1u);
                PROF_MARK(2)
                const double *T5 = htabs + buf * 2 * TBL;
                const double *Td = T5 + TBL;
                const double *Glo = gains, *Ghi = gains + TBL;
                const int pa = A.pairs.a[cur], pb = A.pairs.b[cur], pd = A.pairs.d[cur];
                const bool self = pa == pb;
                bool on[NT][2];
                double we[NT][2];
                const double wu = wts[qg]; // first point of the warp's group
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        on[nt][e] = lnz >> (6 * (2 * nt + e) + pa) & 1u;
                        we[nt][e] = NKRC ? 0.0 : wts[qg + nt * 8 + 2 * lc + e]; // generic paths only
                    }
                // Pressure-weight mode of the warp's 16 points (warp-uniform, set once per
                // half-batch).  Points are compacted in GridState order (j fastest), so a group
                // of 16 almost always sits on one model level and shares one pressure:
                //   0: all w == 0 (p <= 500 hPa): K500 + Kd*0 == K500 exactly -> one half
                //   1: all w == wu: K = K500 + wu*Kd interpolated in the A fragment -> one half
                //   2: otherwise (group straddles a level): K500 half + w * (Kd half)
                const int wmode = wmode_s[wid];
                const double *vbase[2] = {&W(pb, lc, qg + lr), &W(pa, lc, qg + lr)};

                for (int X = 0; X < (self ? 1 : 2); ++X) {
                    const int V = X == 1 ? 2 : (self ? 1 : 0); // gain view
                    const int fcat = X == 0 ? pa : pb;
                    const double *vb = vbase[X];
                    // A-operand addressing: row pass T[o][s], column pass T[s][o]
                    const int o = o0 + lr;
                    const int astride = X == 0 ? 4 : 4 * S;             // per K-step
                    const int abase = X == 0 ? o * S + lc : lc * S + o; // at ks = 0
                    const int kf = F.kf[V][b], km = F.km[V][b];
                    const int kzf = kzg[g][fcat], kzs = kzg[g][X == 0 ? pb : pa];
                    const int kend = (kzs >> 2) + 1; // K-steps that can see a non-zero B
                    if (o0 <= kzf && kzs >= 0) {     // else every product of this block is zero
                    double Y1[NT][2], Y2[NT][2], YG[NT][2];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
                        Y1[nt][0] = Y1[nt][1] = Y2[nt][0] = Y2[nt][1] = YG[nt][0] = YG[nt][1] = 0.0;
                    const int nhalf = wmode == 2 ? 2 : 1;
                    // compiled-in grid: a level-straddling group runs the unrolled dual pass
                    const bool unrolled = NKRC ? true : (F.std_classes && wmode != 2);
                    if (unrolled) { // fully unrolled K-loops (the common case)
                        double c1[NT][2] = {}, c2[NT][2], cg[NT][2];
                        if (NKRC && wmode == 2) {
                            double wqq[NT];
#pragma unroll
                            for (int nt = 0; nt < NT; ++nt) wqq[nt] = wts[qg + 8 * nt + lr];
#define FSBM_PASS2(BB)                                                                             \
    (X == 0 ? dmma_pass_dual<2 * BB, 2 * BB + 2, 9, 4>(T5, Td, wqq, Glo, Ghi, abase, vb, QP, V, o, lc, c1, c2, cg) \
            : dmma_pass_dual<2 * BB, 2 * BB + 2, 9, 4 * 36>(T5, Td, wqq, Glo, Ghi, abase, vb, QP, V, o, lc, c1, c2, cg))
                            switch (b) {
                            case 0: FSBM_PASS2(0); break;
                            case 1: FSBM_PASS2(1); break;
                            case 2: FSBM_PASS2(2); break;
                            default: FSBM_PASS2(3); break;
                            }
#undef FSBM_PASS2
                        } else {
#define FSBM_PASS(BB, IN)                                                                          \
    (X == 0 ? dmma_pass_single<2 * BB, 2 * BB + 2, 9, IN, 4>(T5, Td, wi, Glo, Ghi, abase, astride, vb, QP, V, o, lc, c1, c2, cg) \
            : dmma_pass_single<2 * BB, 2 * BB + 2, 9, IN, 4 * 36>(T5, Td, wi, Glo, Ghi, abase, astride, vb, QP, V, o, lc, c1, c2, cg))
                        // one instantiation per block (K500 + w*Kd with w = 0 for p <= 500 hPa):
                        // halving the unrolled code keeps the kernel inside the instruction cache
                        const double wi = wmode == 1 ? wu : 0.0;
                        if (wmode == 0) { // p <= 500 hPa: A = K500 exactly, no interpolation
                            switch (b) {
                            case 0: FSBM_PASS(0, false); break;
                            case 1: FSBM_PASS(1, false); break;
                            case 2: FSBM_PASS(2, false); break;
                            default: FSBM_PASS(3, false); break;
                            }
                        } else {
                            switch (b) {
                            case 0: FSBM_PASS(0, true); break;
                            case 1: FSBM_PASS(1, true); break;
                            case 2: FSBM_PASS(2, true); break;
                            default: FSBM_PASS(3, true); break;
                            }
                        }
#undef FSBM_PASS
                        }
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                Y1[nt][e] = c1[nt][e];
                                Y2[nt][e] = c2[nt][e];
                                YG[nt][e] = cg[nt][e];
                            }
                    }
                    for (int h = 0; h < (unrolled ? 0 : nhalf); ++h) {
                        const double *Ta = h == 0 ? T5 : Td;
                        const bool summed = wmode == 1;
                        double c1[NT][2], c2[NT][2], cg[NT][2];
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt)
                            c1[nt][0] = c1[nt][1] = c2[nt][0] = c2[nt][1] = 0.0;
                        int ai = abase;
#pragma unroll 2
                        for (int ks = 0; ks < min(kf, kend); ++ks, ai += astride) { // every cell owned-far
                            const double t = summed ? fma(wu, Td[ai], T5[ai]) : Ta[ai];
                            const double t2 = t * Glo[ai];
#pragma unroll
                            for (int nt = 0; nt < NT; ++nt) {
                                const double v = vb[(4 * ks) * QP + nt * 8];
                                dmma(c1[nt][0], c1[nt][1], t, v);
                                dmma(c2[nt][0], c2[nt][1], t2, v);
                            }
                        }
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) { // YG shares the loss DMMAs so far
                            cg[nt][0] = c1[nt][0];
                            cg[nt][1] = c1[nt][1];
                        }
                        for (int ks = kf; ks < min(km, kend); ++ks, ai += astride) { // diagonal steps
                            const int s = 4 * ks + lc;
                            const double t = summed ? fma(wu, Td[ai], T5[ai]) : Ta[ai];
                            // gain view: R-cross s<o, R-self s<o (+ s==o at 1/2), C s<=o
                            const double msk = V == 2 ? (s <= o ? 1.0 : 0.0)
                                                      : (s < o ? 1.0 : (V == 1 && s == o ? 0.5 : 0.0));
                            const int gi = V == 1 && s == o ? o * S + o : ai;
                            const double lo = msk * Glo[gi], hi = msk * Ghi[gi];
                            const double t2 = t * lo, tg = t * (lo + hi);
#pragma unroll
                            for (int nt = 0; nt < NT; ++nt) {
                                const double v = vb[(4 * ks) * QP + nt * 8];
                                dmma(c1[nt][0], c1[nt][1], t, v);
                                dmma(c2[nt][0], c2[nt][1], t2, v);
                                dmma(cg[nt][0], cg[nt][1], tg, v);
                            }
                        }
#pragma unroll 2
                        for (int ks = km; ks < min(KS, kend); ++ks, ai += astride) { // no owned gains
                            const double t = summed ? fma(wu, Td[ai], T5[ai]) : Ta[ai];
#pragma unroll
                            for (int nt = 0; nt < NT; ++nt) {
                                const double v = vb[(4 * ks) * QP + nt * 8];
                                dmma(c1[nt][0], c1[nt][1], t, v);
                            }
                        }
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const double sc = h == 1 ? we[nt][e] : 1.0;
                                Y1[nt][e] = fma(sc, c1[nt][e], Y1[nt][e]);
                                Y2[nt][e] = fma(sc, c2[nt][e], Y2[nt][e]);
                                YG[nt][e] = fma(sc, cg[nt][e], YG[nt][e]);
                            }
                    }
                    PROF_MARK(3)
                    // emission: rows o, points qg+nt*8+2lc+e; hi-gain -> row o+1
                    DmmaAcc L, Gn;
                    DmmaAcc Cy;
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int q = qg + nt * 8 + 2 * lc + e;
                            const double f = on[nt][e] ? W(fcat, o, q) : 0.0; // dt: applied at the apply
                            const double y3 = f * (YG[nt][e] - Y2[nt][e]);
                            const double up = __shfl_up_sync(0xffffffffu, y3, 4);
                            L[nt][e] = f * Y1[nt][e];
                            Gn[nt][e] = lr > 0 ? fma(f, Y2[nt][e], up) : f * Y2[nt][e];
                            Cy[nt][e] = lr == 7 ? y3 : 0.0; // hi gain of row 7 -> next block head
                        }
                    {
                        const uint32_t tf = tmw + 8 * fcat, tp = tmw + 8 * pd, tcy = tmw + 48 + 8 * pd;
                        double d[4], e4[4], cy[4];
                        tm_wait_st(); // the previous emission's stores (long complete by now)
                        tm_ld4_nowait(tf, d);
                        if (fcat != pd) tm_ld4_nowait(tp, e4);
                        tm_ld4_nowait(tcy, cy);
                        tm_wait_ld();
#pragma unroll
                        for (int i = 0; i < 4; ++i) cy[i] += Cy[i >> 1][i & 1];
                        tm_st4_nowait(tcy, cy);
                        if (fcat == pd) {
#pragma unroll
                            for (int i = 0; i < 4; ++i) d[i] += Gn[i >> 1][i & 1] - L[i >> 1][i & 1];
                            tm_st4_nowait(tf, d);
                        } else {
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                d[i] -= L[i >> 1][i & 1];
                                e4[i] += Gn[i >> 1][i & 1];
                            }
                            tm_st4_nowait(tf, d);
                            tm_st4_nowait(tp, e4);
                        }
                    }

                    PROF_MARK(6)
                    } // non-zero block
                    // the top row (bin nkr-1, nkr % 8 == 1): a 1-row GEMM is 1/8 of a DMMA tile, so
                    // it runs on the FP64 CUDA cores, balanced over the group's four warps:
                    // warp b takes points 4b..4b+3 of the group, 8 lanes per point split s.
                    if (TAIL > 0 && kzf >= ot && kzs >= 0) { // top bin non-zero somewhere
                        const int qt = qg + 4 * b + (lane >> 3), sc0 = lane & 7;
                        const double wq = wts[qt];
                        const double *vt = &W(X == 0 ? pb : pa, 0, qt);
                        double y1 = 0.0, y2 = 0.0;
                        if (NKRC) { // columns s < 32 have mask 1 in every view: unrolled, no bound
#pragma unroll
                            for (int r = 0; r < RB; ++r) {
                                const int sx = sc0 + 8 * r;
                                const int ti = X == 0 ? ot * S + sx : sx * S + ot;
                                const double kv = fma(wq, Td[ti], T5[ti]) * vt[static_cast<size_t>(sx) * QP];
                                y1 += kv;
                                y2 = fma(kv, Glo[ti], y2);
                            }
                            if (sc0 == 0 && kzs >= ot) { // s == 32: the view's diagonal weight
                                const int ti = ot * S + ot;
                                const double m = V == 2 ? 1.0 : (V == 1 ? 0.5 : 0.0);
                                const double kv = fma(wq, Td[ti], T5[ti]) * vt[static_cast<size_t>(ot) * QP];
                                y1 += kv;
                                y2 = fma(kv, m * Glo[ti], y2);
                            }
                        } else {
                            for (int sx = sc0; sx <= kzs; sx += 8) {
                                const int ti = X == 0 ? ot * S + sx : sx * S + ot;
                                const double m = V == 2 ? (sx <= ot ? 1.0 : 0.0)
                                                        : (sx < ot ? 1.0 : (V == 1 && sx == ot ? 0.5 : 0.0));
                                const double kv = fma(wq, Td[ti], T5[ti]) * vt[static_cast<size_t>(sx) * QP];
                                y1 += kv;
                                y2 = fma(kv, m * Glo[ti], y2);
                            }
                        }
#pragma unroll
                        for (int d = 1; d < 8; d <<= 1) {
                            y1 += __shfl_xor_sync(0xffffffffu, y1, d);
                            y2 += __shfl_xor_sync(0xffffffffu, y2, d);
                        }
                        if (sc0 == 0 && (act[qt] >> cur & 1ull)) {
                            const double f = W(fcat, ot, qt);
                            tdel[static_cast<size_t>(fcat) * NP + qt] -= f * y1;
                            tdel[static_cast<size_t>(pd) * NP + qt] += f * y2;
                        }
                    }
                }
                PROF_MARK(1)
                // exception cells (non owner-local targets), gathered by the target's owner
                if (!NKRC && F.nexc > 0) { // (the compiled-in 33-bin grid has none)
                    for (int kind = self ? 1 : 0; kind <= (self ? 1 : 2); kind += self ? 1 : 2) {
                        double exd[4] = {0.0, 0.0, 0.0, 0.0};
                        const int T = o0 + lr;
                        const int e0 = __ldg(F.exc_off + kind * (nkr + 1) + T);
                        const int e1 = __ldg(F.exc_off + kind * (nkr + 1) + T + 1);
                        for (int ee = e0; ee < e1; ++ee) {
                            const ExcEntry en = F.exc[ee];
                            const double k5 = T5[static_cast<size_t>(en.i) * S + en.j];
                            const double kd = Td[static_cast<size_t>(en.i) * S + en.j];
#pragma unroll
                            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                                for (int e = 0; e < 2; ++e) {
                                    const int q = qg + nt * 8 + 2 * lc + e;
                                    const double x = fma(we[nt][e], kd, k5) * W(pa, en.i, q) * W(pb, en.j, q);
                                    if (on[nt][e]) exd[2 * nt + e] += en.coef * x;
                                }
                        }
                        if (__any_sync(0xffffffffu, e1 > e0)) {
                            double d[4];
                            tm_wait_st();
                            tm_ld4_nowait(tmw + 8 * pd, d);
                            tm_wait_ld();
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                d[i] += exd[i];
                                exd[i] = 0.0;
                            }
                            tm_st4_nowait(tmw + 8 * pd, d);
                            tm_wait_st();
                        }
                        if (TAIL > 0 && (lane & 7) == 0) { // targets in the top row: the scalar
                            const int qt = qg + 4 * b + (lane >> 3); // top row's point split
                            const int e2 = __ldg(F.exc_off + kind * (nkr + 1) + ot);
                            const int e3 = __ldg(F.exc_off + kind * (nkr + 1) + ot + 1);
                            for (int ee = e2; ee < e3; ++ee) {
                                const ExcEntry en = F.exc[ee];
                                const double k5 = T5[static_cast<size_t>(en.i) * S + en.j];
                                const double kd = Td[static_cast<size_t>(en.i) * S + en.j];
                                const double x = fma(wts[qt], kd, k5) * W(pa, en.i, qt) * W(pb, en.j, qt);
                                if (act[qt] >> cur & 1ull) tdel[static_cast<size_t>(pd) * NP + qt] += en.coef * x;
                            }
                        }
                    }
                }
                // release buffer `buf`; the last warp of the half refills it with pair n+NBUF
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();
                    const int old = atomicAdd(&relcnt[h][buf], 1);
                    if (old == NWH - 1) {
                        relcnt[h][buf] = 0;
                        __threadfence_block();
                        int p2 = nxt; // pair n + NBUF
                        for (int i = 1; i < NBUF; ++i) p2 = next_pair(p2);
                        if (p2 >= 0) {
                            fence_proxy_async();
                            mbar_expect_tx(&hbar[buf], tbytes);
                            tma_bulk_g2s(htabs + buf * 2 * TBL, F.blob + static_cast<size_t>(p2) * 2 * TBL,
                                         tbytes, &hbar[buf]);
                        }
                    }
                }
                cur = nxt;
                ++n;
            }
            pbase += n;
            PROF_MARK(7)
            // ---- Jacobi apply (coalescence.cpp:313-328): every read of `work` for this
            // substep (in this half) is done.  Phase 1: each warp adds its TMEM deltas to its
            // own 8 rows and parks the hi-gain carry of its row 7 (TMEM) for the next block's
            // head in the half's idle table ring (block 3's goes to the top row via tdel).
            // Phase 2: block heads take the carry, the top row takes tdel, and each warp checks
            // the rows it owns for negative values (no clamping; every failing bin of a
            // point is offered, the sink keeps the first in serial order).
            half_sync(h);
            PROF_MARK(4)
            const bool prefetch = sub == A.substeps - 1 && htid < NPH;
            uint32_t pf_p = 0xffffffffu; // the next half-batch's points, loaded early
            double pf_w = 0.0;
            if (prefetch) fetch_point(hb + kDmmaH * gridDim.x, pf_p, pf_w);
            double *cscr = htabs; // [6][RB-1][NP] carry scratch (the ring is idle here)
            double nv[kNCat][4];
            tm_wait_st();
            {
                double d[kNCat][4];
#pragma unroll
                for (int c = 0; c < kNCat; ++c) tm_ld4_nowait(tmw + 8 * c, d[c]);
                tm_wait_ld();
#pragma unroll
                for (int c = 0; c < kNCat; ++c)
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int q = qg + (i >> 1) * 8 + 2 * lc + (i & 1);
                        nv[c][i] = fma(dt, d[c][i], W(c, o0 + lr, q));
                        W(c, o0 + lr, q) = nv[c][i];
                    }
            }
            {
                double cy[kNCat][4];
#pragma unroll
                for (int c = 0; c < kNCat; ++c) tm_ld4_nowait(tmw + 48 + 8 * c, cy[c]);
                tm_wait_ld();
                if (lr == 7) {
#pragma unroll
                    for (int c = 0; c < kNCat; ++c)
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int q = qg + (i >> 1) * 8 + 2 * lc + (i & 1);
                            if (b + 1 < RB) cscr[(static_cast<size_t>(c) * (RB - 1) + b) * NP + q] = cy[c][i];
                            else if (TAIL > 0) tdel[static_cast<size_t>(c) * NP + q] += cy[c][i];
                        }
                }
            }
            half_sync(h);
            if (b > 0 && lr == 0) { // block head: the previous block's carry
#pragma unroll
                for (int c = 0; c < kNCat; ++c)
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int q = qg + (i >> 1) * 8 + 2 * lc + (i & 1);
                        nv[c][i] = fma(dt, cscr[(static_cast<size_t>(c) * (RB - 1) + b - 1) * NP + q], nv[c][i]);
                        W(c, o0, q) = nv[c][i];
                    }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) { // the first failing category of each of the lane's points
                int cf = -1;
                double vf = 0.0;
#pragma unroll
                for (int c = kNCat - 1; c >= 0; --c)
                    if (nv[c][i] < 0.0) {
                        cf = c;
                        vf = nv[c][i];
                    }
                if (cf >= 0) {
                    const int q = qg + (i >> 1) * 8 + 2 * lc + (i & 1);
                    const uint32_t p = pidx[q];
                    if (p != 0xffffffffu && (pfail[q] & 1) == 0) {
                        report_stiffness(A, p, cf, o0 + lr, vf);
                        atomicOr(&pfail[q], 2); // bit 1: concurrent writers, bit 0 gates
                    }
                }
            }
            if (TAIL > 0 && b == RB - 1) // the top row of this group's 16 points
                for (int f = lane; f < kNCat * NT * 8; f += 32) {
                    const int c = f / (NT * 8), q = qg + f % (NT * 8);
                    const double v = fma(dt, tdel[static_cast<size_t>(c) * NP + q], W(c, ot, q));
                    W(c, ot, q) = v;
                    const uint32_t p = pidx[q];
                    if (v < 0.0 && p != 0xffffffffu && (pfail[q] & 1) == 0) {
                        report_stiffness(A, p, c, ot, v);
                        atomicOr(&pfail[q], 2); // bit 1: concurrent writers, bit 0 gates
                    }
                }
            if (prefetch) {
                nx_p[q0 + htid] = pf_p;
                nx_w[q0 + htid] = pf_w;
            }
            half_sync(h);
            if (htid < NPH && pfail[q0 + htid] == 2) pfail[q0 + htid] = 3;
        }
        // ---- write back + counters ----
        {
            constexpr int NQ = kNCat * NPH / 4;
            const int qs = lane >> 3, kc = lane & 7;
            for (int u = hwid; u < NQ; u += NWH) {
                const int c = u / (NPH / 4), q = q0 + 4 * (u % (NPH / 4)) + qs;
                const uint32_t p = pidx[q];
                if (p == 0xffffffffu) continue;
                double *dst = A.bins[c] + static_cast<size_t>(p) * nkr;
#pragma unroll
                for (int jj = 0; jj < 5; ++jj) {
                    const int k = kc + 8 * jj;
                    if (k < nkr) dst[k] = W(c, k, q);
                }
            }
        }
        if (htid < NPH) {
            const int q = q0 + htid;
            if (pidx[q] != 0xffffffffu && pfail[q] == 0) {
                tr_acc += ptrip[q];
                pt_acc += 1;
                ev_acc += A.kernel_strategy ? ptrip[q] : full_evals;
            }
        }
        half_sync(h);
        PROF_MARK(5)
    }
    PROF_FLUSH
    tm_fence_before();
    __syncthreads();
    if (wid == 0) {
        tm_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
    for (int o = 16; o > 0; o >>= 1) {
        tr_acc += __shfl_down_sync(0xffffffffu, tr_acc, o);
        pt_acc += __shfl_down_sync(0xffffffffu, pt_acc, o);
        ev_acc += __shfl_down_sync(0xffffffffu, ev_acc, o);
    }
    if (lane == 0 && (tr_acc | pt_acc | ev_acc)) {
        atomicAdd(&A.counters[0], tr_acc);
        atomicAdd(&A.counters[1], pt_acc);
        atomicAdd(&A.counters[2], ev_acc);
    }
}

inline size_t dmma_smem_bytes(int nkr, int S, int QP) {
    constexpr int NP = kDmmaNP;
    const size_t TBL = static_cast<size_t>(S) * S;
    const size_t d = (2 * kDmmaH * kDmmaNBUF + 2) * TBL + static_cast<size_t>(kNCat) * S * QP +
                     static_cast<size_t>(kNCat) * NP + NP;
    return d * 8 + NP * 8 * 2 + (kDmmaH * kDmmaNBUF + 1) * 8 + NP * 4 + NP * 4;
}

/// Returns -1 when this geometry cannot run the DMMA path (caller falls back).
inline int launch_dmma(const DmmaTables &T, const FastTables & /*FT*/, const StepArgs &A,
                       int num_sms, cudaStream_t s) {
    if (!T.blob || A.nkr != T.nkr) return -1;
    const int QP = kDmmaQP;
    const size_t smem = dmma_smem_bytes(A.nkr, T.S, QP);
    if (smem > 227 * 1024) return -1;
    DmmaArgs F{};
    F.S = T.S;
    F.tail = A.nkr % 8;
    F.QP = QP;
    for (int V = 0; V < 3; ++V)
        for (int b = 0; b < kDmmaRB; ++b) {
            F.kf[V][b] = T.kf[V][b];
            F.km[V][b] = T.km[V][b];
        }
    F.std_classes = T.S == 36;
    for (int V = 0; V < 3; ++V)
        for (int b = 0; b < kDmmaRB; ++b)
            F.std_classes = F.std_classes && T.kf[V][b] == 2 * b && T.km[V][b] == 2 * b + 2;
    if (const char *ev = std::getenv("FSBM_DMMA_UNROLL"); ev && ev[0] == '0') F.std_classes = 0; // A/B
    F.nbatches = (A.nactive_host + kDmmaNPH - 1) / kDmmaNPH; // 32-point half-batches
    F.blob = T.blob;
    F.gains = T.gains;
    F.exc_off = T.exc_off;
    F.exc = T.exc;
    F.nexc = T.nexc;
    const bool c33 = A.nkr == 33 && F.std_classes && T.nexc == 0 && !std::getenv("FSBM_DMMA_GENERIC");
    auto kern = c33 ? coal_dmma_kernel<33> : coal_dmma_kernel<0>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess) {
        fast_err() = "dmma path: cannot reserve shared memory";
        return 6;
    }
    const int grid = static_cast<int>(std::min<uint32_t>((F.nbatches + kDmmaH - 1) / kDmmaH, num_sms));
#ifdef FSBM_DMMA_PROF
    constexpr int kPW = kDmmaThreads / 32; // warps per CTA
    static unsigned long long *dprof = nullptr;
    if (!dprof) {
        cudaMalloc(&dprof, kPW * 8 * 8);
        cudaMemset(dprof, 0, kPW * 8 * 8);
    }
    F.prof = dprof;
#endif
    kern<<<grid, kDmmaThreads, smem, s>>>(A, F);
#ifdef FSBM_DMMA_PROF
    {
        unsigned long long h[kPW * 8];
        cudaStreamSynchronize(s);
        cudaMemcpy(h, dprof, sizeof(h), cudaMemcpyDeviceToHost);
        static int calls = 0;
        if (++calls % 4 == 0) {
            fprintf(stderr, "dmma prof (Gcycles per warp, all CTAs): setup tail wait kloops barrier rest emit other\n");
            for (int w = 0; w < kPW; ++w) {
                fprintf(stderr, "  w%2d b%d:", w, (w % 4 + w / 4) % 4);
                for (int k = 0; k < 8; ++k) fprintf(stderr, " %7.2f", h[w * 8 + k] / 1e9);
                fprintf(stderr, "\n");
            }
        }
    }
#endif
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fast_err() = std::string("dmma path launch: ") + cudaGetErrorString(e);
        return 6;
    }
    return 0;
}

} // namespace fsbm
