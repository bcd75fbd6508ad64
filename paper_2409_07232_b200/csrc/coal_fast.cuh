// coal_fast.cuh -- FSBM_NUMERICS_FAST: the throughput path for coal_step on sm_100a.
//
// Same mathematics as coal_step (proj/src/coalescence.cpp:204-339) with the sums
// reassociated so that every accumulation is owned by one thread (deterministic,
// no atomics on values, bitwise reproducible run to run):
//
//   rate(i,j) = K(i,j) na[i] nb[j],  K = K500 + w (K750-K500)   (kernels.hpp:123-135)
//   loss_a[i] = na[i] dt  sum_j K(i,j) nb[j]        -- "row pass": owner = row i
//   loss_b[j] = nb[j] dt  sum_i K(i,j) na[i]        -- "column pass": owner = column j
//   gain[lo]  += dn w_lo, gain[lo+1] += dn w_hi     -- Kovetz-Olund split (GainTable)
//
// The gain of a cell below the diagonal (j < i) lands in bins (i, i+1) for almost
// every cell (flux target lo = max(i,j), measured 79-91% of cells), so the row
// owner accumulates it in two registers; cells on/above the diagonal land in
// (j, j+1) and are owned by the column pass.  The remaining "exception" cells
// (near-diagonal lo > max(i,j), and top-bin-rule cells whose target is not the
// owner) are gathered per target bin from a host-built CSR list.  Self pairs use
// the symmetrised table K(min(i,j), max(i,j)) over the full square in a single
// row pass: its row sums are the reference's total loss of bin i (row i plus
// column i of the j>=i triangle), and each below-diagonal cell stands for its
// mirrored reference cell, so the triangle walk folds onto a balanced rectangle.
//
// Thread geometry: a warp is R row-slots x (32/R) point groups, each thread holds
// P=2 points, so one 16-byte table load feeds 2*(32/R) point-cells and the
// per-point spectrum operand of a step is a broadcast shared-memory load.  A CTA
// holds one or more "sets" of 2*(32/R) points whose spectra/deltas live in smem.
#pragma once

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "fsbm_common.cuh"

namespace fsbm {

struct ExcEntry {
    int i, j;
    double coef;
};

struct FastTables {
    int nkr = 0, npairs = 0;
    double2 *TR = nullptr; // [pair][t=j][r=i]  (K500, Kd) for the row pass (self: symmetrised/2)
    double2 *TC = nullptr; // [pair][t=i][r=j]  (K500, Kd) raw, column pass + exceptions
    double2 *GR = nullptr; // [t=j][r=i] (c_lo, c_hi) owner-local gains of the row pass
    double2 *GC = nullptr; // [t=i][r=j] (c_lo, c_hi) owner-local gains of the column pass
    int *exc_off = nullptr;      // [3][nkr+1]: 0 row-pass cross, 1 row-pass self, 2 column pass
    ExcEntry *exc = nullptr;     // entries referenced by exc_off
    int exc_max = 0;
};

inline std::string &fast_err() {
    static thread_local std::string e;
    return e;
}
inline const char *fast_last_error() { return fast_err().c_str(); }

inline void free_fast_tables(FastTables &f) {
    cudaFree(f.TR);
    cudaFree(f.TC);
    cudaFree(f.GR);
    cudaFree(f.GC);
    cudaFree(f.exc_off);
    cudaFree(f.exc);
    f = FastTables{};
}

/// Host-side preparation of the pass-ordered tables (point-independent, done once).
inline int build_fast_tables(FastTables &f, int nkr, const std::vector<double> & /*x*/,
                             int npairs, const std::vector<int> &abd, const double *t750,
                             const double *t500, const std::vector<int32_t> &g_lo,
                             const std::vector<double> &g_wlo, const std::vector<double> &g_whi,
                             const std::vector<double> &g_top) {
    const size_t nn = static_cast<size_t>(nkr) * nkr;
    std::vector<double2> TR(npairs * nn), TC(npairs * nn), GR(nn, double2{0, 0}),
        GC(nn, double2{0, 0});
    for (int p = 0; p < npairs; ++p) {
        const bool self = abd[3 * p] == abd[3 * p + 1];
        const double *k750 = t750 + p * nn, *k500 = t500 + p * nn;
        for (int i = 0; i < nkr; ++i)
            for (int j = 0; j < nkr; ++j) {
                const size_t e = static_cast<size_t>(i) * nkr + j;
                const double kd = k750[e] - k500[e];
                TC[p * nn + e] = double2{k500[e], kd}; // [t=i][r=j]
                double r500 = k500[e], rkd = kd;
                if (self) { // reference reads only j >= i: K_sym(i,j) = K(min,max)
                    const size_t u = static_cast<size_t>(std::min(i, j)) * nkr + std::max(i, j);
                    r500 = k500[u];
                    rkd = k750[u] - k500[u];
                }
                TR[p * nn + static_cast<size_t>(j) * nkr + i] = double2{r500, rkd}; // [t=j][r=i]
            }
    }
    // owner-local gain coefficients + exception lists (per target bin)
    std::vector<std::vector<ExcEntry>> ex[3];
    for (auto &v : ex) v.assign(nkr, {});
    // Self-pair entries are stored as (min,max): the reference reads only the
    // j >= i triangle, and na == nb so the product is unchanged.
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
            const size_t e = static_cast<size_t>(i) * nkr + j;
            const int lo = g_lo[e];
            if (j < i) { // below the diagonal: row pass owns the gain (owner i)
                if (lo == i) {
                    GR[static_cast<size_t>(j) * nkr + i] = double2{g_wlo[e], g_whi[e]};
                } else if (lo < 0 && i == nkr - 1) {
                    GR[static_cast<size_t>(j) * nkr + i] = double2{g_top[e], 0.0};
                } else {
                    add_exc(0, i, j, 1.0);
                    add_exc(1, i, j, 1.0);
                }
            } else { // on/above the diagonal: column pass owns it (owner j)
                if (lo == j) {
                    GC[static_cast<size_t>(i) * nkr + j] = double2{g_wlo[e], g_whi[e]};
                } else if (lo < 0 && j == nkr - 1) {
                    GC[static_cast<size_t>(i) * nkr + j] = double2{g_top[e], 0.0};
                } else {
                    add_exc(2, i, j, 1.0);
                }
                if (i == j) add_exc(1, i, i, 0.5); // self diagonal: rate halved (coalescence.cpp:293)
            }
        }
    std::vector<int> off(3 * (nkr + 1));
    std::vector<ExcEntry> all;
    int mx = 0;
    for (int k = 0; k < 3; ++k) {
        for (int t = 0; t < nkr; ++t) {
            off[k * (nkr + 1) + t] = static_cast<int>(all.size());
            all.insert(all.end(), ex[k][t].begin(), ex[k][t].end());
            mx = std::max<int>(mx, static_cast<int>(ex[k][t].size()));
        }
        off[k * (nkr + 1) + nkr] = static_cast<int>(all.size());
    }
    if (all.empty()) all.push_back({0, 0, 0.0});
    auto up = [](auto **dst, const auto &v) {
        using T = typename std::remove_reference<decltype(v)>::type::value_type;
        if (cudaMalloc(reinterpret_cast<void **>(dst), sizeof(T) * v.size()) != cudaSuccess)
            return false;
        return cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice) ==
               cudaSuccess;
    };
    f.nkr = nkr;
    f.npairs = npairs;
    f.exc_max = mx;
    if (!up(&f.TR, TR) || !up(&f.TC, TC) || !up(&f.GR, GR) || !up(&f.GC, GC) ||
        !up(&f.exc_off, off) || !up(&f.exc, all)) {
        fast_err() = "fast tables: device allocation failed";
        return 6;
    }
    return 0;
}

struct FastArgs {
    int nsets;   // point sets per CTA
    int rounds;  // row rounds per pass
    int npts;    // points per CTA batch
    uint32_t nbatches;
    double2 const *TR, *TC, *GR, *GC;
    int const *exc_off;
    ExcEntry const *exc;
};

template <int R> struct FastGeom {
    static constexpr int Q = 32 / R; // point groups per warp
    static constexpr int P = 2;      // points per thread
    static constexpr int PTS = Q * P;
};

constexpr int kFastWarps = 17;

__device__ inline double sel(bool on, double v) { return on ? v : 0.0; }

template <int R>
__global__ void __launch_bounds__(kFastWarps * 32, 1)
    coal_fast_kernel(StepArgs A, FastArgs F) {
    using G = FastGeom<R>;
    constexpr int PTS = G::PTS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nkr = A.nkr;
    const int nsets = F.nsets;
    const size_t arr = static_cast<size_t>(nsets) * kNCat * nkr * PTS; // doubles per buffer
    double *work = reinterpret_cast<double *>(smem_raw);
    double *delta = work + arr;
    double *dhi = delta + arr;
    double *wts = dhi + arr;                                     // [npts]
    unsigned long long *act = reinterpret_cast<unsigned long long *>(wts + F.npts); // [npts]
    unsigned long long *ptrip = act + F.npts;                    // [npts]
    uint32_t *pidx = reinterpret_cast<uint32_t *>(ptrip + F.npts); // [npts]
    int *pfail = reinterpret_cast<int *>(pidx + F.npts);         // [npts]
    // last non-zero bin per (point, category): products with an exactly-zero spectrum value
    // vanish (the reference skips rate == 0 triples, coalescence.cpp:286-292), so a row's
    // stream loop stops there and a row whose owner values are zero skips its emission
    short *lz = reinterpret_cast<short *>(pfail + F.npts);        // [npts][6]
    __shared__ unsigned long long cta_act;

    auto IX = [&](int s, int c, int k, int q) -> size_t {
        return ((static_cast<size_t>(s) * kNCat + c) * nkr + k) * PTS + q;
    };

    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int rsub = lane % R, grp = lane / R;
    const int V = kFastWarps * R; // row slots per round
    if (A.stale && *A.stale) return; // stale mask: the step must not touch the state
    const uint32_t nact = *A.nactive;
    const int npairs = A.pairs.npairs;
    const unsigned long long full_evals = static_cast<unsigned long long>(npairs) * nkr * nkr;
    const int self_tri = nkr * (nkr + 1) / 2, cross_sq = nkr * nkr;

    unsigned long long tr_acc = 0, pt_acc = 0, ev_acc = 0;

    for (uint32_t batch = blockIdx.x; batch < F.nbatches && batch * static_cast<uint32_t>(F.npts) < nact;
         batch += gridDim.x) {
        // ---- load the batch: point ids, weights, spectra --------------------
        for (int q = tid; q < F.npts; q += nthr) {
            const uint32_t idx = batch * static_cast<uint32_t>(F.npts) + q;
            const bool live = idx < nact;
            const uint32_t p = live ? A.active[idx] : 0xffffffffu;
            pidx[q] = p;
            wts[q] = live ? pressure_weight(A.pressure[p]) : 0.0;
            pfail[q] = live ? 0 : 1;
            ptrip[q] = 0;
        }
        __syncthreads();
        {
            const int tot = nsets * kNCat * nkr * PTS;
            for (int f = tid; f < tot; f += nthr) { // q fastest: conflict-free smem stores
                const int q = f % PTS;
                int rest = f / PTS;
                const int k = rest % nkr;
                rest /= nkr;
                const int c = rest % kNCat;
                const int s = rest / kNCat;
                const uint32_t p = pidx[s * PTS + q];
                work[IX(s, c, k, q)] =
                    p != 0xffffffffu ? A.bins[c][static_cast<size_t>(p) * nkr + k] : 0.0;
            }
        }
        for (int sub = 0; sub < A.substeps; ++sub) {
            // ---- zero deltas, pair-activity (all_zero, coalescence.cpp:270-273) ----
            for (size_t f = tid; f < 2 * arr; f += nthr) delta[f] = 0.0;
            if (tid == 0) cta_act = 0ull;
            __syncthreads();
            for (int q = tid; q < F.npts; q += nthr) {
                const int s = q / PTS, qq = q % PTS;
                unsigned nz = 0;
                for (int c = 0; c < kNCat; ++c) { // scanned from the top: last non-zero bin
                    int l = nkr - 1;
                    while (l >= 0 && work[IX(s, c, l, qq)] == 0.0) --l;
                    nz |= l >= 0 ? (1u << c) : 0u;
                    lz[q * kNCat + c] = static_cast<short>(l);
                }
                unsigned long long m = 0;
                unsigned long long trip = 0;
                for (int pp = 0; pp < npairs; ++pp)
                    if (nz >> A.pairs.a[pp] & 1u) {
                        m |= 1ull << pp;
                        trip += A.pairs.a[pp] == A.pairs.b[pp] ? self_tri : cross_sq;
                    }
                if (pfail[q] == 0) {
                    act[q] = m;
                    atomicOr(&cta_act, m);
                    ptrip[q] += trip; // counted only if the point succeeds (coalescence.cpp:333-338)
                } else {
                    act[q] = 0;
                }
            }
            __syncthreads();
            const unsigned long long amask = cta_act;

            for (int pp = 0; pp < npairs; ++pp) {
                if (!(amask >> pp & 1ull)) continue;
                const int a = A.pairs.a[pp], b = A.pairs.b[pp], d = A.pairs.d[pp];
                const bool self = a == b;
                const double2 *TRp = F.TR + static_cast<size_t>(pp) * nkr * nkr;
                const double2 *TCp = F.TC + static_cast<size_t>(pp) * nkr * nkr;
                for (int rd = 0; rd < F.rounds; ++rd) {
                    const int vr = rd * V + warp * R + rsub;
                    const int s = vr / nkr, r = vr % nkr;
                    if (s >= nsets) continue; // idle slot (no barrier inside the pass)
                    const int q0 = grp * 2;
                    const bool on0 = act[s * PTS + q0] >> pp & 1ull;
                    const bool on1 = act[s * PTS + q0 + 1] >> pp & 1ull;
                    const double w0 = wts[s * PTS + q0], w1 = wts[s * PTS + q0 + 1];
                    const double *na = work + IX(s, a, 0, q0);
                    const double *nb = work + IX(s, b, 0, q0);
                    // row pass (owner row r, stream nb[t]) and column pass (owner col r, stream na[t])
                    double accR0 = 0, accR1 = 0, alR0 = 0, alR1 = 0, ahR0 = 0, ahR1 = 0;
                    double accC0 = 0, accC1 = 0, alC0 = 0, alC1 = 0, ahC0 = 0, ahC1 = 0;
                    const double2 nar = *reinterpret_cast<const double2 *>(na + static_cast<size_t>(r) * PTS);
                    const double2 nbr = *reinterpret_cast<const double2 *>(nb + static_cast<size_t>(r) * PTS);
                    const short *l0 = lz + (s * PTS + q0) * kNCat, *l1 = l0 + kNCat;
                    // stream bins past the last non-zero one contribute nothing
                    const int tend = 1 + max(max(l0[a], l0[b]), max(l1[a], l1[b]));
                    const bool live_row = nar.x != 0.0 || nar.y != 0.0 || (!self && (nbr.x != 0.0 || nbr.y != 0.0));
                    if (!live_row) {
                        // every owner term of this row is zero; exceptions below still run
                    } else if (self) {
#pragma unroll 4
                        for (int t = 0; t < tend; ++t) {
                            const double2 kk = __ldg(TRp + static_cast<size_t>(t) * nkr + r);
                            const double2 gc = __ldg(F.GR + static_cast<size_t>(t) * nkr + r);
                            const double2 sv = *reinterpret_cast<const double2 *>(nb + static_cast<size_t>(t) * PTS);
                            const double k0 = fma(w0, kk.y, kk.x), k1 = fma(w1, kk.y, kk.x);
                            const double t0 = k0 * sv.x, t1 = k1 * sv.y;
                            accR0 += t0;
                            accR1 += t1;
                            alR0 = fma(t0, gc.x, alR0);
                            alR1 = fma(t1, gc.x, alR1);
                            ahR0 = fma(t0, gc.y, ahR0);
                            ahR1 = fma(t1, gc.y, ahR1);
                        }
                    } else {
#pragma unroll 2
                        for (int t = 0; t < tend; ++t) {
                            const double2 kr = __ldg(TRp + static_cast<size_t>(t) * nkr + r);
                            const double2 gr = __ldg(F.GR + static_cast<size_t>(t) * nkr + r);
                            const double2 kc = __ldg(TCp + static_cast<size_t>(t) * nkr + r);
                            const double2 gc = __ldg(F.GC + static_cast<size_t>(t) * nkr + r);
                            const double2 sb = *reinterpret_cast<const double2 *>(nb + static_cast<size_t>(t) * PTS);
                            const double2 sa = *reinterpret_cast<const double2 *>(na + static_cast<size_t>(t) * PTS);
                            const double kr0 = fma(w0, kr.y, kr.x), kr1 = fma(w1, kr.y, kr.x);
                            const double kc0 = fma(w0, kc.y, kc.x), kc1 = fma(w1, kc.y, kc.x);
                            const double tr0 = kr0 * sb.x, tr1 = kr1 * sb.y;
                            const double tc0 = kc0 * sa.x, tc1 = kc1 * sa.y;
                            accR0 += tr0;
                            accR1 += tr1;
                            alR0 = fma(tr0, gr.x, alR0);
                            alR1 = fma(tr1, gr.x, alR1);
                            ahR0 = fma(tr0, gr.y, ahR0);
                            ahR1 = fma(tr1, gr.y, ahR1);
                            accC0 += tc0;
                            accC1 += tc1;
                            alC0 = fma(tc0, gc.x, alC0);
                            alC1 = fma(tc1, gc.x, alC1);
                            ahC0 = fma(tc0, gc.y, ahC0);
                            ahC1 = fma(tc1, gc.y, ahC1);
                        }
                    }
                    // ---- owner emission: delta[*][r] (owner r), dhi[d][r+1] (owner r) ----
                    const double fR0 = nar.x * A.dt_sub, fR1 = nar.y * A.dt_sub;
                    double *dA = delta + IX(s, a, r, q0);
                    double *dD = delta + IX(s, d, r, q0);
                    dA[0] -= sel(on0, fR0 * accR0);
                    dA[1] -= sel(on1, fR1 * accR1);
                    dD[0] += sel(on0, fR0 * alR0);
                    dD[1] += sel(on1, fR1 * alR1);
                    if (r + 1 < nkr) {
                        double *hD = dhi + IX(s, d, r + 1, q0);
                        hD[0] += sel(on0, fR0 * ahR0);
                        hD[1] += sel(on1, fR1 * ahR1);
                    }
                    if (!self) {
                        const double fC0 = nbr.x * A.dt_sub, fC1 = nbr.y * A.dt_sub;
                        double *dB = delta + IX(s, b, r, q0);
                        dB[0] -= sel(on0, fC0 * accC0);
                        dB[1] -= sel(on1, fC1 * accC1);
                        dD[0] += sel(on0, fC0 * alC0);
                        dD[1] += sel(on1, fC1 * alC1);
                        if (r + 1 < nkr) {
                            double *hD = dhi + IX(s, d, r + 1, q0);
                            hD[0] += sel(on0, fC0 * ahC0);
                            hD[1] += sel(on1, fC1 * ahC1);
                        }
                    }
                    // ---- exception cells whose gain targets bin r (gathered by owner r) ----
                    for (int kind = self ? 1 : 0; kind <= (self ? 1 : 2); kind += self ? 1 : 2) {
                        const int *off = F.exc_off + kind * (nkr + 1);
                        const int e0 = __ldg(off + r), e1 = __ldg(off + r + 1);
                        double x0 = 0.0, x1 = 0.0;
                        for (int e = e0; e < e1; ++e) {
                            const ExcEntry ee = F.exc[e];
                            const double2 kk = __ldg(TCp + static_cast<size_t>(ee.i) * nkr + ee.j);
                            const double2 ai = *reinterpret_cast<const double2 *>(na + static_cast<size_t>(ee.i) * PTS);
                            const double2 bj = *reinterpret_cast<const double2 *>(nb + static_cast<size_t>(ee.j) * PTS);
                            const double k0 = fma(w0, kk.y, kk.x), k1 = fma(w1, kk.y, kk.x);
                            x0 = fma(ee.coef, k0 * ai.x * bj.x, x0);
                            x1 = fma(ee.coef, k1 * ai.y * bj.y, x1);
                        }
                        dD[0] += sel(on0, x0 * A.dt_sub);
                        dD[1] += sel(on1, x1 * A.dt_sub);
                    }
                }
            }
            __syncthreads();
            // ---- Jacobi apply + stiffness (coalescence.cpp:313-328), write back ----
            {
                const int tot = nsets * kNCat * nkr * PTS;
                for (int f = tid; f < tot; f += nthr) {
                    const int q = f % PTS;
                    int rest = f / PTS;
                    const int k = rest % nkr;
                    rest /= nkr;
                    const int c = rest % kNCat;
                    const int s = rest / kNCat;
                    const int qi = s * PTS + q;
                    const uint32_t p = pidx[qi];
                    if (p == 0xffffffffu) continue;
                    const size_t ix = IX(s, c, k, q);
                    const double v = work[ix] + (delta[ix] + dhi[ix]);
                    work[ix] = v;
                    // every failing bin is offered (the sink keeps the first in serial
                    // order); bit 1 marks the failing substep, only bit 0 gates (set at barriers)
                    if (v < 0.0 && (pfail[qi] & 1) == 0) {
                        report_stiffness(A, p, c, k, v);
                        atomicOr(&pfail[qi], 2); // first failing substep marks the point
                    }
                }
            }
            __syncthreads();
            for (int q = tid; q < F.npts; q += nthr)
                if (pfail[q] == 2) pfail[q] = 3; // freeze after the failing substep
        }
        // ---- write back + counters ----------------------------------------
        {
            const int tot = nsets * kNCat * nkr * PTS;
            for (int f = tid; f < tot; f += nthr) {
                const int q = f % PTS;
                int rest = f / PTS;
                const int k = rest % nkr;
                rest /= nkr;
                const int c = rest % kNCat;
                const int s = rest / kNCat;
                const uint32_t p = pidx[s * PTS + q];
                if (p != 0xffffffffu)
                    A.bins[c][static_cast<size_t>(p) * nkr + k] = work[IX(s, c, k, q)];
            }
        }
        for (int q = tid; q < F.npts; q += nthr) {
            if (pidx[q] == 0xffffffffu || pfail[q] != 0) continue; // failing points throw first
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
    if (lane == 0) {
        atomicAdd(&A.counters[0], tr_acc);
        atomicAdd(&A.counters[1], pt_acc);
        atomicAdd(&A.counters[2], ev_acc);
    }
}

inline size_t fast_smem_bytes(int nkr, int nsets, int pts) {
    const size_t arr = static_cast<size_t>(nsets) * kNCat * nkr * pts;
    const size_t npts = static_cast<size_t>(nsets) * pts;
    return 3 * arr * sizeof(double) + npts * (sizeof(double) + 8 + 8 + 4 + 4 + kNCat * sizeof(short));
}

template <int R>
inline int launch_fast_r(const FastTables &T, const StepArgs &A, int num_sms, cudaStream_t s) {
    using G = FastGeom<R>;
    const int V = kFastWarps * R;
    FastArgs F{};
    F.nsets = std::max(1, V / A.nkr);
    F.rounds = (F.nsets * A.nkr + V - 1) / V;
    F.npts = F.nsets * G::PTS;
    F.nbatches = (A.nactive_host + F.npts - 1) / F.npts;
    F.TR = T.TR;
    F.TC = T.TC;
    F.GR = T.GR;
    F.GC = T.GC;
    F.exc_off = T.exc_off;
    F.exc = T.exc;
    size_t smem = fast_smem_bytes(A.nkr, F.nsets, G::PTS);
    while (smem > 200 * 1024 && F.nsets > 1) {
        F.nsets -= 1;
        F.rounds = (F.nsets * A.nkr + V - 1) / V;
        F.npts = F.nsets * G::PTS;
        F.nbatches = (A.nactive_host + F.npts - 1) / F.npts;
        smem = fast_smem_bytes(A.nkr, F.nsets, G::PTS);
    }
    if (smem > 227 * 1024) {
        fast_err() = "fast path: nkr=" + std::to_string(A.nkr) + " needs " +
                     std::to_string(smem) + " bytes of shared memory";
        return 5;
    }
    if (cudaFuncSetAttribute(coal_fast_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess) {
        fast_err() = "fast path: cannot reserve shared memory";
        return 6;
    }
    const int grid = static_cast<int>(std::min<uint32_t>(F.nbatches, num_sms));
    coal_fast_kernel<R><<<grid, kFastWarps * 32, smem, s>>>(A, F);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fast_err() = std::string("fast path launch: ") + cudaGetErrorString(e);
        return 6;
    }
    return 0;
}

/// Chooses the row-slot geometry so a CTA's point state fits in shared memory.
inline int launch_fast(const FastTables &T, const StepArgs &A, int num_sms, cudaStream_t s) {
    if (A.nkr <= 80) return launch_fast_r<4>(T, A, num_sms, s);
    if (A.nkr <= 160) return launch_fast_r<8>(T, A, num_sms, s);
    return launch_fast_r<16>(T, A, num_sms, s);
}

} // namespace fsbm
