// coal_dmma.cuh -- FSBM_NUMERICS_FAST on the FP64 tensor cores (DMMA.8x8x4), nkr <= 40.
//
// Same reassociated mathematics as coal_fast.cuh (row pass / column pass, owner-
// local Kovetz-Olund gains, exception gather), restated as small GEMMs over a
// batch of points so that the FP64 tensor pipe does the multiply-adds:
//
//   pass X (X = row: owner o = i, stream s = j, v = nb, f = na;
//           X = col: owner o = j, stream s = i, v = na, f = nb):
//     Y_k[o,q] = sum_s (P_k^500[o,s] + w_q P_k^d[o,s]) v_q[s],   k = 1 (loss), 2 (lo), 3 (hi)
//     P_1 = T_X, P_2 = T_X * clo_X, P_3 = T_X * chi_X           (T_X = K500 / K750-K500)
//   => per (pass, product): C[o, q] += A[o, s] B[s, q] with A = P_k (8 rows x 4 s per
//      DMMA) and B = [v ; w*v] (4 s x 8 points), K-dim = both halves of s.
//   emission: delta[src][o] -= dt f Y1,  delta[d][o] += dt f Y2,  delta[d][o+1] += dt f Y3.
//
// Work split: warp (g, b) owns rows o in [8b, 8b+8) for the NT*8 points of group g,
// for every pair, pass and product, so its deltas live in registers (no atomics,
// deterministic); the hi-gain of row 8b+7 is carried to the next block through
// smem.  Rows beyond the last full 8-row block (the "tail", e.g. the top bin at
// 33 bins) are done in direct FP64 by one extra warp.  Per-pair tables (row and
// column layouts, 4 x nkr x S doubles) are double-buffered in smem by a 1-D TMA
// bulk copy (cp.async.bulk + mbarrier) issued one pair ahead.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "coal_fast.cuh"
#include "fsbm_common.cuh"

namespace fsbm {

struct DmmaTables {
    int nkr = 0, S = 0, npairs = 0;
    int kf[2][8] = {}, km[2][8] = {}; // see DmmaArgs
    double *blob = nullptr;  // [pair][TR500 | TRd | TC500 | TCd], each [nkr][S], zero padded
    double *gains = nullptr; // [GRlo | GRhi | GClo | GChi], each [nkr][S]
};

inline void free_dmma_tables(DmmaTables &t) {
    cudaFree(t.blob);
    cudaFree(t.gains);
    t = DmmaTables{};
}

constexpr int kDmmaMaxNkr = 40;

inline int build_dmma_tables(DmmaTables &D, int nkr, int npairs, const std::vector<int> &abd,
                             const double *t750, const double *t500,
                             const std::vector<int32_t> &g_lo, const std::vector<double> &g_wlo,
                             const std::vector<double> &g_whi, const std::vector<double> &g_top) {
    if (nkr > kDmmaMaxNkr || nkr < 8) return 0; // path unused for this grid
    const int S = (nkr + 3) / 4 * 4;
    const size_t nn = static_cast<size_t>(nkr) * S;
    std::vector<double> blob(static_cast<size_t>(npairs) * 4 * nn, 0.0), gains(4 * nn, 0.0);
    const size_t sq = static_cast<size_t>(nkr) * nkr;
    for (int p = 0; p < npairs; ++p) {
        const bool self = abd[3 * p] == abd[3 * p + 1];
        const double *k750 = t750 + p * sq, *k500 = t500 + p * sq;
        double *b = blob.data() + static_cast<size_t>(p) * 4 * nn;
        for (int i = 0; i < nkr; ++i)
            for (int j = 0; j < nkr; ++j) {
                const size_t e = static_cast<size_t>(i) * nkr + j;
                const size_t u = self ? static_cast<size_t>(std::min(i, j)) * nkr + std::max(i, j) : e;
                b[0 * nn + static_cast<size_t>(i) * S + j] = k500[u];           // row pass [o=i][s=j]
                b[1 * nn + static_cast<size_t>(i) * S + j] = k750[u] - k500[u];
                b[2 * nn + static_cast<size_t>(j) * S + i] = k500[e];           // col pass [o=j][s=i]
                b[3 * nn + static_cast<size_t>(j) * S + i] = k750[e] - k500[e];
            }
    }
    for (int i = 0; i < nkr; ++i)
        for (int j = 0; j < nkr; ++j) {
            const size_t e = static_cast<size_t>(i) * nkr + j;
            const int lo = g_lo[e];
            if (j < i) { // row pass owns it (owner i): same rule as coal_fast.cuh
                double clo = 0, chi = 0;
                if (lo == i) { clo = g_wlo[e]; chi = g_whi[e]; }
                else if (lo < 0 && i == nkr - 1) { clo = g_top[e]; }
                gains[0 * nn + static_cast<size_t>(i) * S + j] = clo;
                gains[1 * nn + static_cast<size_t>(i) * S + j] = chi;
            } else { // column pass (owner j)
                double clo = 0, chi = 0;
                if (lo == j) { clo = g_wlo[e]; chi = g_whi[e]; }
                else if (lo < 0 && j == nkr - 1) { clo = g_top[e]; }
                gains[2 * nn + static_cast<size_t>(j) * S + i] = clo;
                gains[3 * nn + static_cast<size_t>(j) * S + i] = chi;
            }
        }
    // K-step classification per pass / 8-row block (prefix structure of owned far cells)
    const int KS = S / 4;
    for (int X = 0; X < 2; ++X)
        for (int b = 0; b < nkr / 8 && b < 8; ++b) {
            const double *glo = gains.data() + (2 * X) * nn, *ghi = glo + nn;
            auto cls = [&](int ks) { // 0 all far-owned (clo+chi==1), 2 all zero, 1 mixed
                bool all_one = true, all_zero = true;
                for (int r = 0; r < 8; ++r)
                    for (int c = 0; c < 4; ++c) {
                        const size_t ix = static_cast<size_t>(8 * b + r) * S + 4 * ks + c;
                        const double sum = glo[ix] + ghi[ix];
                        all_one = all_one && std::fabs(sum - 1.0) <= 4e-16;
                        all_zero = all_zero && glo[ix] == 0.0 && ghi[ix] == 0.0;
                    }
                return all_one ? 0 : all_zero ? 2 : 1;
            };
            int kf = 0;
            while (kf < KS && cls(kf) == 0) ++kf;
            int km = KS;
            while (km > kf && cls(km - 1) == 2) --km;
            D.kf[X][b] = kf;
            D.km[X][b] = km;
        }
    D.nkr = nkr;
    D.S = S;
    D.npairs = npairs;
    if (cudaMalloc(&D.blob, blob.size() * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&D.gains, gains.size() * sizeof(double)) != cudaSuccess ||
        cudaMemcpy(D.blob, blob.data(), blob.size() * sizeof(double), cudaMemcpyHostToDevice) !=
            cudaSuccess ||
        cudaMemcpy(D.gains, gains.data(), gains.size() * sizeof(double), cudaMemcpyHostToDevice) !=
            cudaSuccess) {
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
/// D(8x8) += A(8x4) B(4x8), FP64 tensor core.
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

struct DmmaArgs {
    int S, RB, tail;      // padded stream length, full 8-row blocks, tail rows
    int kf[2][8], km[2][8]; // per pass/block: leading all-owned-far K-steps, end of gain K-steps
    int QP;               // smem point pitch (>= NP, = 4 mod 16)
    uint32_t nbatches;
    const double *blob, *gains;
    const int *exc_off;
    const ExcEntry *exc;
};

template <int NT> struct DmmaGeom {
    static constexpr int G = 3;                // point groups per CTA
    static constexpr int NP = G * NT * 8;      // points per batch
};

/// register delta add with a runtime (warp-uniform) category
template <int NT>
__device__ __forceinline__ void dadd_cat(double (&D)[kNCat][NT][2], int cat, int nt, int e,
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

template <int NT>
__global__ void __launch_bounds__(384, 1)
    coal_dmma_kernel(StepArgs A, DmmaArgs F) {
    constexpr int G = DmmaGeom<NT>::G;
    constexpr int NP = DmmaGeom<NT>::NP;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nkr = A.nkr, S = F.S, RB = F.RB, QP = F.QP, TAIL = F.tail;
    const size_t TBL = static_cast<size_t>(nkr) * S; // doubles per table
    double *tabs = reinterpret_cast<double *>(smem_raw);         // [2][4][nkr][S]
    double *gains = tabs + 8 * TBL;                               // [4][nkr][S]
    double *work = gains + 4 * TBL;                               // [6][S][QP]
    double *carry = work + static_cast<size_t>(kNCat) * S * QP;   // [6][RB][NP]
    double *tdel = carry + static_cast<size_t>(kNCat) * RB * NP;  // [6][TAIL][NP]
    double *wts = tdel + static_cast<size_t>(kNCat) * std::max(TAIL, 1) * NP; // [NP]
    unsigned long long *act = reinterpret_cast<unsigned long long *>(wts + NP);  // [NP]
    unsigned long long *ptrip = act + NP;                                        // [NP]
    uint64_t *mbar = reinterpret_cast<uint64_t *>(ptrip + NP);                   // [3]
    uint32_t *pidx = reinterpret_cast<uint32_t *>(mbar + 3);                     // [NP]
    int *pfail = reinterpret_cast<int *>(pidx + NP);                             // [NP]
    double *dstage = tabs; // [6][nkr][NP] at substep end (tables are idle then)
    __shared__ unsigned long long cta_act;
    __shared__ int relcnt[2];

    const int tid = threadIdx.x, nthr = blockDim.x;
    const int wid = tid >> 5, lane = tid & 31;
    const bool is_mma = wid < G * RB;
    // block b of group g: rotate by g so each SMSP (wid % 4) hosts a mix of blocks
    // (the lower-triangular gain work grows with b)
    const int g = is_mma ? wid / RB : 0, b = is_mma ? (wid % RB + g) % RB : 0;
    const int NW = nthr >> 5;
    const int o0 = 8 * b;
    const int lr = lane >> 2, lc = lane & 3;
    const uint32_t nact = *A.nactive;
    const int npairs = A.pairs.npairs;
    const unsigned long long full_evals = static_cast<unsigned long long>(npairs) * nkr * nkr;
    const int self_tri = nkr * (nkr + 1) / 2, cross_sq = nkr * nkr;
    const double dt = A.dt_sub;
    unsigned long long tr_acc = 0, pt_acc = 0, ev_acc = 0;

    auto W = [&](int c, int s, int q) -> double & {
        return work[(static_cast<size_t>(c) * S + s) * QP + q];
    };

    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        mbar_init(&mbar[2], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) { // pair-independent gain coefficients, once per CTA
        mbar_expect_tx(&mbar[2], static_cast<uint32_t>(4 * TBL * sizeof(double)));
        tma_bulk_g2s(gains, F.gains, static_cast<uint32_t>(4 * TBL * sizeof(double)), &mbar[2]);
    }
    uint32_t use[2] = {0u, 0u}; // completed phases per table buffer (uniform across threads)
    bool gains_ready = false;

    for (uint32_t batch = blockIdx.x; batch < F.nbatches; batch += gridDim.x) {
        for (int q = tid; q < NP; q += nthr) {
            const uint32_t idx = batch * static_cast<uint32_t>(NP) + q;
            const bool live = idx < nact;
            const uint32_t p = live ? A.active[idx] : 0xffffffffu;
            pidx[q] = p;
            wts[q] = live ? pressure_weight(A.pressure[p]) : 0.0;
            pfail[q] = live ? 0 : 1;
            ptrip[q] = 0;
        }
        __syncthreads();
        for (int c = 0; c < kNCat; ++c) // q across lanes: conflict-free STS
            for (int k = wid; k < S; k += NW)
                for (int q = lane; q < NP; q += 32) {
                    const uint32_t p = pidx[q];
                    W(c, k, q) = (p != 0xffffffffu && k < nkr) ? A.bins[c][static_cast<size_t>(p) * nkr + k] : 0.0;
                }
        if (!gains_ready) {
            mbar_wait(&mbar[2], 0);
            gains_ready = true;
        }
        __syncthreads();

        for (int sub = 0; sub < A.substeps; ++sub) {
            if (tid == 0) cta_act = 0ull;
            for (int f = tid; f < kNCat * (RB + std::max(TAIL, 1)) * NP; f += nthr) carry[f] = 0.0;
            __syncthreads();
            for (int q = tid; q < NP; q += nthr) { // all_zero (coalescence.cpp:270-273)
                unsigned nz = 0;
                for (int c = 0; c < kNCat; ++c) {
                    bool any = false;
                    for (int k = 0; k < nkr && !any; ++k) any = W(c, k, q) != 0.0;
                    nz |= any ? (1u << c) : 0u;
                }
                unsigned long long m = 0, trip = 0;
                for (int pp = 0; pp < npairs; ++pp)
                    if (nz >> A.pairs.a[pp] & 1u) {
                        m |= 1ull << pp;
                        trip += A.pairs.a[pp] == A.pairs.b[pp] ? self_tri : cross_sq;
                    }
                if (pfail[q] == 0) {
                    act[q] = m;
                    atomicOr(&cta_act, m);
                    ptrip[q] += trip;
                } else {
                    act[q] = 0;
                }
            }
            __syncthreads();
            const unsigned long long amask = cta_act;

            double D[kNCat][NT][2];
#pragma unroll
            for (int c = 0; c < kNCat; ++c)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) D[c][nt][0] = D[c][nt][1] = 0.0;

            // Pair pipeline without CTA barriers: tables of pairs n and n+1 are in flight
            // in the two buffers; the LAST warp to release buffer (n&1) issues the TMA of
            // pair n+2 into it, so warps drift and one warp's emission overlaps another
            // warp's DMMAs.  full = mbar[buf] (TMA transaction), empty = relcnt[buf].
            auto next_pair = [&](int p) -> int {
                if (p < 0) return -1;
                const unsigned long long rest = amask & ~((2ull << p) - 1ull);
                return rest ? __ffsll(static_cast<long long>(rest)) - 1 : -1;
            };
            const uint32_t tbytes = static_cast<uint32_t>(4 * TBL * sizeof(double));
            int cur = amask ? __ffsll(static_cast<long long>(amask)) - 1 : -1;
            int n = 0;
            if (tid == 0) {
                relcnt[0] = relcnt[1] = 0;
                fence_proxy_async(); // dstage (generic writes) -> TMA overwrite
                if (cur >= 0) {
                    mbar_expect_tx(&mbar[0], tbytes);
                    tma_bulk_g2s(tabs, F.blob + static_cast<size_t>(cur) * 4 * TBL, tbytes, &mbar[0]);
                }
                const int p1 = next_pair(cur);
                if (p1 >= 0) {
                    mbar_expect_tx(&mbar[1], tbytes);
                    tma_bulk_g2s(tabs + 4 * TBL, F.blob + static_cast<size_t>(p1) * 4 * TBL, tbytes, &mbar[1]);
                }
            }
            __syncthreads();
            while (cur >= 0) {
                const int buf = n & 1;
                const int nxt = next_pair(cur);
                mbar_wait(&mbar[buf], use[buf] & 1u);
                use[buf] += 1;
                const double *tb = tabs + buf * 4 * TBL;
                const int pa = A.pairs.a[cur], pb = A.pairs.b[cur], pd = A.pairs.d[cur];
                const bool self = pa == pb;

                if (is_mma) {
                    const int qg = g * NT * 8;
                    // per-lane activity of this pair for the emission points
                    bool on[NT][2];
                    double we[NT][2];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int q = qg + nt * 8 + 2 * lc + e;
                            on[nt][e] = act[q] >> cur & 1ull;
                            we[nt][e] = wts[q];
                        }
                    // Pressure-weight mode of this warp's 16 points (warp-uniform):
                    //   0: all w == 0 (p <= 500 hPa)  -> K500 + Kd*0 == K500 exactly: one half
                    //   1: all w == 1 (p >= 750 hPa)  -> K = K500 + Kd (the same sum the
                    //      reference forms): one half on the summed table
                    //   2: otherwise                   -> K500 half + w * (Kd half)
                    bool all0 = true, all1 = true;
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            all0 = all0 && we[nt][e] == 0.0;
                            all1 = all1 && we[nt][e] == 1.0;
                        }
                    const int wmode = __all_sync(0xffffffffu, all0) ? 0 : __all_sync(0xffffffffu, all1) ? 1 : 2;
                    for (int X = 0; X < (self ? 1 : 2); ++X) {
                        const double *T5 = tb + (2 * X) * TBL;
                        const double *Td = T5 + TBL;
                        const double *Glo = gains + (2 * X) * TBL;
                        const double *Ghi = Glo + TBL;
                        const int vcat = X == 0 ? pb : pa; // stream category
                        const int fcat = X == 0 ? pa : pb; // owner scale / loss category
                        const int kf = F.kf[X][b], km = F.km[X][b], KS = S / 4;
                        // Y1 = loss sum, Y2 = lo-gain sum, YG = sum of T*(clo+chi) v, so
                        // Y3 (hi-gain) = YG - Y2.  In the leading K-steps every cell of the
                        // block is an owned far cell (clo+chi == 1), so YG reuses the loss DMMAs
                        // there; only the diagonal ("mixed") steps need an explicit T*(clo+chi).
                        double Y1[NT][2], Y2[NT][2], YG[NT][2];
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt)
                            Y1[nt][0] = Y1[nt][1] = Y2[nt][0] = Y2[nt][1] = YG[nt][0] = YG[nt][1] = 0.0;
                        const size_t arow = static_cast<size_t>(o0 + lr) * S + lc;
                        const double *vb = &W(vcat, lc, qg + lr);
                        const int nhalf = wmode == 2 ? 2 : 1;
                        for (int h = 0; h < nhalf; ++h) {
                            // h == 0: K500 (mode 0/2) or K500+Kd (mode 1); h == 1: Kd (mode 2)
                            const double *Ta = (h == 0) ? T5 : Td;
                            const bool summed = wmode == 1;
                            double c1o[NT][2], c1r[NT][2], c2[NT][2], cg[NT][2];
#pragma unroll
                            for (int nt = 0; nt < NT; ++nt)
                                c1o[nt][0] = c1o[nt][1] = c1r[nt][0] = c1r[nt][1] = c2[nt][0] = c2[nt][1] =
                                    cg[nt][0] = cg[nt][1] = 0.0;
#pragma unroll 2
                            for (int ks = 0; ks < kf; ++ks) { // owned far cells only
                                const size_t ai = arow + 4 * ks;
                                const double t = summed ? T5[ai] + Td[ai] : Ta[ai];
                                const double t2 = t * Glo[ai];
#pragma unroll
                                for (int nt = 0; nt < NT; ++nt) {
                                    const double v = vb[static_cast<size_t>(4 * ks) * QP + nt * 8];
                                    dmma(c1o[nt][0], c1o[nt][1], t, v);
                                    dmma(c2[nt][0], c2[nt][1], t2, v);
                                }
                            }
                            for (int ks = kf; ks < km; ++ks) { // diagonal / mixed steps
                                const size_t ai = arow + 4 * ks;
                                const double t = summed ? T5[ai] + Td[ai] : Ta[ai];
                                const double lo = Glo[ai];
                                const double t2 = t * lo, tg = t * (lo + Ghi[ai]);
#pragma unroll
                                for (int nt = 0; nt < NT; ++nt) {
                                    const double v = vb[static_cast<size_t>(4 * ks) * QP + nt * 8];
                                    dmma(c1r[nt][0], c1r[nt][1], t, v);
                                    dmma(c2[nt][0], c2[nt][1], t2, v);
                                    dmma(cg[nt][0], cg[nt][1], tg, v);
                                }
                            }
#pragma unroll 2
                            for (int ks = km; ks < KS; ++ks) { // no gains owned by this pass
                                const size_t ai = arow + 4 * ks;
                                const double t = summed ? T5[ai] + Td[ai] : Ta[ai];
#pragma unroll
                                for (int nt = 0; nt < NT; ++nt) {
                                    const double v = vb[static_cast<size_t>(4 * ks) * QP + nt * 8];
                                    dmma(c1r[nt][0], c1r[nt][1], t, v);
                                }
                            }
#pragma unroll
                            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                                for (int e = 0; e < 2; ++e) {
                                    const double sc = h == 1 ? we[nt][e] : 1.0;
                                    Y1[nt][e] = fma(sc, c1o[nt][e] + c1r[nt][e], Y1[nt][e]);
                                    Y2[nt][e] = fma(sc, c2[nt][e], Y2[nt][e]);
                                    YG[nt][e] = fma(sc, c1o[nt][e] + cg[nt][e], YG[nt][e]);
                                }
                        }
                        // emission (owner rows o0+lr, points qg+nt*8+2lc+e)
                        const int o = o0 + lr;
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const int q = qg + nt * 8 + 2 * lc + e;
                                const double f = on[nt][e] ? W(fcat, o, q) * dt : 0.0;
                                const double y1 = f * Y1[nt][e];
                                const double y2 = f * Y2[nt][e];
                                const double y3 = f * (YG[nt][e] - Y2[nt][e]);
                                const double up = __shfl_up_sync(0xffffffffu, y3, 4);
                                dadd_cat<NT>(D, fcat, nt, e, -y1);
                                dadd_cat<NT>(D, pd, nt, e, lr > 0 ? y2 + up : y2);
                                if (lr == 7) carry[(static_cast<size_t>(pd) * RB + b) * NP + q] += y3;
                            }
                    }
                    // exceptions targeting my rows (gathered by the owner lane)
                    for (int kind = self ? 1 : 0; kind <= (self ? 1 : 2); kind += self ? 1 : 2) {
                        const int T = o0 + lr;
                        const int e0 = __ldg(F.exc_off + kind * (nkr + 1) + T);
                        const int e1 = __ldg(F.exc_off + kind * (nkr + 1) + T + 1);
                        for (int ee = e0; ee < e1; ++ee) {
                            const ExcEntry en = F.exc[ee];
                            const double k5 = tb[static_cast<size_t>(en.i) * S + en.j];
                            const double kd = tb[TBL + static_cast<size_t>(en.i) * S + en.j];
#pragma unroll
                            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                                for (int e = 0; e < 2; ++e) {
                                    const int q = qg + nt * 8 + 2 * lc + e;
                                    const double kw = fma(we[nt][e], kd, k5);
                                    const double x = kw * W(pa, en.i, q) * W(pb, en.j, q);
                                    if (on[nt][e]) dadd_cat<NT>(D, pd, nt, e, en.coef * x * dt);
                                }
                        }
                    }
                }
                // tail rows o in [8RB, nkr), direct FP64: 8 lanes per point split the
                // stream sum (fixed-order xor reduction -> deterministic)
                if (TAIL > 0 && tid < NP * 8) {
                    const int q = tid >> 3, sl = tid & 7;
                    const bool onq = act[q] >> cur & 1ull;
                    const double w = wts[q];
                    for (int X = 0; X < (self ? 1 : 2); ++X) {
                        const double *T5 = tb + (2 * X) * TBL;
                        const double *Td = T5 + TBL;
                        const double *Glo = gains + (2 * X) * TBL;
                        const double *Ghi = Glo + TBL;
                        const int vcat = X == 0 ? pb : pa;
                        const int fcat = X == 0 ? pa : pb;
                        for (int t = 0; t < TAIL; ++t) {
                            const int o = 8 * RB + t;
                            double y1 = 0, y2 = 0, y3 = 0;
                            for (int s2 = sl; s2 < nkr; s2 += 8) {
                                const size_t ai = static_cast<size_t>(o) * S + s2;
                                const double kw = fma(w, Td[ai], T5[ai]);
                                const double tt = kw * W(vcat, s2, q);
                                y1 += tt;
                                y2 = fma(tt, Glo[ai], y2);
                                y3 = fma(tt, Ghi[ai], y3);
                            }
#pragma unroll
                            for (int m = 1; m < 8; m <<= 1) {
                                y1 += __shfl_xor_sync(0xffffffffu, y1, m);
                                y2 += __shfl_xor_sync(0xffffffffu, y2, m);
                                y3 += __shfl_xor_sync(0xffffffffu, y3, m);
                            }
                            if (sl == 0 && onq) {
                                const double f = W(fcat, o, q) * dt;
                                tdel[(static_cast<size_t>(fcat) * TAIL + t) * NP + q] -= f * y1;
                                tdel[(static_cast<size_t>(pd) * TAIL + t) * NP + q] += f * y2;
                                if (t + 1 < TAIL)
                                    tdel[(static_cast<size_t>(pd) * TAIL + t + 1) * NP + q] += f * y3;
                            }
                        }
                    }
                    if (sl == 0 && onq) {
                        for (int kind = self ? 1 : 0; kind <= (self ? 1 : 2); kind += self ? 1 : 2)
                            for (int t = 0; t < TAIL; ++t) {
                                const int T = 8 * RB + t;
                                const int e0 = __ldg(F.exc_off + kind * (nkr + 1) + T);
                                const int e1 = __ldg(F.exc_off + kind * (nkr + 1) + T + 1);
                                double x = 0.0;
                                for (int ee = e0; ee < e1; ++ee) {
                                    const ExcEntry en = F.exc[ee];
                                    const double kw = fma(w, tb[TBL + static_cast<size_t>(en.i) * S + en.j],
                                                          tb[static_cast<size_t>(en.i) * S + en.j]);
                                    x = fma(en.coef, kw * W(pa, en.i, q) * W(pb, en.j, q), x);
                                }
                                tdel[(static_cast<size_t>(pd) * TAIL + t) * NP + q] += x * dt;
                            }
                    }
                }
                // release buffer `buf`; the last warp out refills it with pair n+2
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();
                    const int old = atomicAdd(&relcnt[buf], 1);
                    if (old == NW - 1) {
                        relcnt[buf] = 0;
                        __threadfence_block();
                        const int p2 = next_pair(nxt);
                        if (p2 >= 0) {
                            fence_proxy_async();
                            mbar_expect_tx(&mbar[buf], tbytes);
                            tma_bulk_g2s(tabs + buf * 4 * TBL, F.blob + static_cast<size_t>(p2) * 4 * TBL,
                                         tbytes, &mbar[buf]);
                        }
                    }
                }
                cur = nxt;
                ++n;
            }
            __syncthreads(); // every warp is done with the last tables before dstage reuses them
            // ---- combine deltas into dstage[c][o][q] (tables are idle now) ----
            if (is_mma) {
                const int qg = g * NT * 8;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int q = qg + nt * 8 + 2 * lc + e;
                        const int o = o0 + lr;
#pragma unroll
                        for (int c = 0; c < kNCat; ++c) {
                            double v = D[c][nt][e];
                            if (lr == 0 && b > 0) v += carry[(static_cast<size_t>(c) * RB + b - 1) * NP + q];
                            dstage[(static_cast<size_t>(c) * nkr + o) * NP + q] = v;
                        }
                    }
            }
            __syncthreads();
            {
                for (int f = tid; f < kNCat * TAIL * NP; f += nthr) {
                    const int q = f % NP;
                    const int t = (f / NP) % TAIL;
                    const int c = f / (NP * TAIL);
                    double v = tdel[f];
                    if (t == 0 && RB > 0) v += carry[(static_cast<size_t>(c) * RB + RB - 1) * NP + q];
                    dstage[(static_cast<size_t>(c) * nkr + 8 * RB + t) * NP + q] = v;
                }
            }
            __syncthreads();
            // ---- Jacobi apply + stiffness (coalescence.cpp:313-328) ----
            for (int c = 0; c < kNCat; ++c)
                for (int k = wid; k < nkr; k += NW)
                    for (int q = lane; q < NP; q += 32) {
                        const uint32_t p = pidx[q];
                        if (p == 0xffffffffu) continue;
                        const double v = W(c, k, q) + dstage[(static_cast<size_t>(c) * nkr + k) * NP + q];
                        W(c, k, q) = v;
                        if (v < 0.0 && pfail[q] == 0) {
                            report_stiffness(A, p, c, k);
                            pfail[q] = 2;
                        }
                    }
            __syncthreads();
            for (int q = tid; q < NP; q += nthr)
                if (pfail[q] == 2) pfail[q] = 3;
            for (int f = tid; f < kNCat * std::max(TAIL, 1) * NP; f += nthr) tdel[f] = 0.0;
            __syncthreads();
        }
        // ---- write back + counters ----
        for (int c = 0; c < kNCat; ++c)
            for (int k = wid; k < nkr; k += NW)
                for (int q = lane; q < NP; q += 32) {
                    const uint32_t p = pidx[q];
                    if (p != 0xffffffffu) A.bins[c][static_cast<size_t>(p) * nkr + k] = W(c, k, q);
                }
        for (int q = tid; q < NP; q += nthr) {
            if (pidx[q] == 0xffffffffu || pfail[q] != 0) continue;
            tr_acc += ptrip[q];
            pt_acc += 1;
            ev_acc += A.kernel_strategy ? ptrip[q] : full_evals;
        }
        __syncthreads();
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

template <int NT>
inline size_t dmma_smem_bytes(int nkr, int S, int RB, int tail, int QP) {
    constexpr int NP = DmmaGeom<NT>::NP;
    const size_t TBL = static_cast<size_t>(nkr) * S;
    size_t d = 8 * TBL + 4 * TBL + static_cast<size_t>(kNCat) * S * QP +
               static_cast<size_t>(kNCat) * RB * NP + static_cast<size_t>(kNCat) * std::max(tail, 1) * NP + NP;
    size_t bytes = d * 8 + NP * 8 * 2 + 3 * 8 + NP * 4 + NP * 4;
    return bytes;
}

/// Returns -1 when this geometry cannot run the DMMA path (caller falls back).
inline int launch_dmma(const DmmaTables &T, const FastTables &FT, const StepArgs &A, int num_sms,
                       cudaStream_t s) {
    constexpr int NT = 2;
    constexpr int NP = DmmaGeom<NT>::NP;
    if (!T.blob || A.nkr != T.nkr) return -1;
    const int S = T.S, RB = A.nkr / 8, tail = A.nkr % 8;
    const int QP = (NP + 15) / 16 * 16 + 4;
    // the substep-end delta stage reuses the two table buffers
    if (static_cast<size_t>(kNCat) * A.nkr * NP > 8 * static_cast<size_t>(A.nkr) * S) return -1;
    const size_t smem = dmma_smem_bytes<NT>(A.nkr, S, RB, tail, QP);
    if (smem > 227 * 1024 || DmmaGeom<NT>::G * RB * 32 > 384 || NP * 8 > DmmaGeom<NT>::G * RB * 32) return -1;
    DmmaArgs F{};
    F.S = S;
    F.RB = RB;
    for (int X = 0; X < 2; ++X)
        for (int b = 0; b < 8; ++b) {
            F.kf[X][b] = T.kf[X][b];
            F.km[X][b] = T.km[X][b];
        }
    F.tail = tail;
    F.QP = QP;
    F.nbatches = (A.nactive_host + NP - 1) / NP;
    F.blob = T.blob;
    F.gains = T.gains;
    F.exc_off = FT.exc_off;
    F.exc = FT.exc;
    const int threads = DmmaGeom<NT>::G * RB * 32;
    if (cudaFuncSetAttribute(coal_dmma_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess) {
        fast_err() = "dmma path: cannot reserve shared memory";
        return 6;
    }
    const int grid = static_cast<int>(std::min<uint32_t>(F.nbatches, num_sms));
    coal_dmma_kernel<NT><<<grid, threads, smem, s>>>(A, F);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fast_err() = std::string("dmma path launch: ") + cudaGetErrorString(e);
        return 6;
    }
    return 0;
}

} // namespace fsbm
