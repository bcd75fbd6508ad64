// coal_bott.cuh -- FSBM_NUMERICS_BOTT: Bott's (1998) flux method on device.
//
// SURVEY 8(f) rank 4 ("coal_bott_new"-style remap).  The reference coalbench splits
// every collision product over two bins by Kovetz-Olund (coalescence.cpp:36-67) and
// declares Bott's flux-form scheme a deliberate divergence; this kernel
// offers it as a third numerics mode behind the same fissioned_step boundary, with the
// same inputs (registry order, interpolated K500/K750 tables, halved self diagonal,
// all_zero skip, GainTable flux target and top rule, counters).  The algorithm and its
// known-answer pinning are in oracle/bott_oracle.c (the checker): per point, on mass per
// bin g = n x, a Gauss-Seidel sweep over pairs, i, j moves z = min(K dt g_a g_b,
// g_a x_j, g_b x_i) out of the two source bins into the target bin k, then Bott's
// exponential sub-grid flux (eq. 13, written with expm1 so it does not cancel) carries
// a share into bin k+1.  Positive-definite: no StiffnessError.
//
// One thread = one mask-true point (the sweep is sequential per point); the 32 lanes of
// a warp walk the same (pair, i, j) in lockstep, so table, gain-target and Courant loads
// are warp-uniform broadcasts.  The point's 6 x nkr masses live in a per-warp global arena
// [category][bin][lane] (one 256-byte line per access, L1/L2-resident): the sweep is a
// long dependent chain per point, so what pays is the number of points in flight -- 32
// warps per SM through the arena measured 3.2x the throughput of a shared-memory state
// (which fits only 4 warps of 33-bin points per SM).  Every product/sum is rounded
// separately (__dmul_rn/__dadd_rn, no FMA) in the oracle's order; only log/log1p/exp/
// expm1 come from CUDA's libdevice instead of glibc (<= 1-2 ulp apart), hence a
// tolerance rather than bitwise parity (tests/test_gpu_bott.py).
#pragma once

#include "fsbm_common.cuh"

namespace fsbm {

constexpr int kBottThreads = 128;
constexpr double kBottLnGmin = -138.15510557964274; // ln(1e-60): Bott's g_min floor

struct BottArgs {
    const double *cour; // [i][j] Courant numbers of the GainTable targets (0 for top cells)
    const double *x;    // [nkr] mass grid
    const double *rx;   // [nkr] 1 / x
    double *arena;      // per-warp [6][nkr][32] point states
};

/// Bott's eq. 13 flux of gsk from bin k (holding gk after the gain) into bin k+1 (gkp),
/// operation for operation as orc_bott_flux (oracle/bott_oracle.c).
__device__ __forceinline__ double bott_flux(double gsk, double gk, double gkp, double c) {
    const double q = __ddiv_rn(1.0, gk), u = __dmul_rn(__dsub_rn(gkp, gk), q), r = __dmul_rn(gkp, q);
    double x1 = (u > -0.5 && u < 0.5) ? log1p(u) : log(__dadd_rn(r, 1e-60));
    if (x1 < kBottLnGmin) x1 = kBottLnGmin;
    if (x1 > -kBottLnGmin) x1 = -kBottLnGmin;
    double flux;
    if (x1 == 0.0) flux = __dmul_rn(gsk, c);
    else
        flux = __ddiv_rn(__dmul_rn(__dmul_rn(gsk, exp(__dmul_rn(x1, __dsub_rn(0.5, c)))), expm1(__dmul_rn(x1, c))), x1);
    return flux < gsk ? flux : gsk;
}

#ifndef FSBM_BOTT_MINB
#define FSBM_BOTT_MINB 8 // 64 registers: 8 blocks (32 warps) per SM, +3% over 80 registers (A/B)
#endif
__global__ void __launch_bounds__(kBottThreads, FSBM_BOTT_MINB) coal_bott_kernel(StepArgs A, BottArgs B) {
    if (A.stale && *A.stale) return; // stale mask: the step must not touch the state
    const int nkr = A.nkr;
    const uint32_t nact = *A.nactive;
    const int lane = threadIdx.x & 31;
    constexpr int L = 32; // stride between a point's values (lanes of one warp interleaved)
    const size_t gwarp = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    double *G = B.arena + gwarp * static_cast<size_t>(kNCat * nkr * 32) + lane;
    const int npairs = A.pairs.npairs;
    const unsigned long long full_evals = static_cast<unsigned long long>(npairs) * nkr * nkr;
    const double dts = A.dt_sub;
    unsigned long long tr_acc = 0, pt_acc = 0, ev_acc = 0;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < nact; base += stride) {
        const uint32_t idx = base + lane;
        const bool live = idx < nact;
        const uint32_t p = live ? A.active[idx] : 0u;
        const double w = live ? pressure_weight(A.pressure[p]) : 0.0;
        for (int c = 0; c < kNCat; ++c) { // masses g = n x
            const double *src = A.bins[c] + static_cast<size_t>(p) * nkr;
            for (int k = 0; k < nkr; ++k)
                G[(c * nkr + k) * L] = live ? __dmul_rn(src[k], __ldg(B.x + k)) : 0.0;
        }
        unsigned long long tr = 0;
        for (int s = 0; s < A.substeps; ++s) {
            for (int q = 0; q < npairs; ++q) {
                const int a = A.pairs.a[q], b = A.pairs.b[q], d = A.pairs.d[q];
                const bool self = a == b;
                double *ga = G + a * nkr * L, *gb = G + b * nkr * L, *gd = G + d * nkr * L;
                bool any = false; // all_zero (coalescence.cpp:270-273), on the current state
                for (int k = 0; k < nkr && !any; ++k) any = ga[k * L] != 0.0;
                if (!any) continue;
                for (int i = 0; i < nkr; ++i) {
                    const int j0 = self ? i : 0;
                    const double *k5 = A.k500 + (static_cast<size_t>(q) * nkr + i) * nkr;
                    const double *kd = A.kd + (static_cast<size_t>(q) * nkr + i) * nkr;
                    const int32_t *glo = A.g_lo + static_cast<size_t>(i) * nkr;
                    const double *cr = B.cour + static_cast<size_t>(i) * nkr;
                    const double xi = __ldg(B.x + i), rxi = __ldg(B.rx + i);
                    for (int j = j0; j < nkr; ++j) {
                        const double gai = ga[i * L], gbj = gb[j * L];
                        if (gai == 0.0 || gbj == 0.0) continue;
                        const bool diagonal = self && i == j;
                        const double xj = __ldg(B.x + j), rxj = __ldg(B.rx + j);
                        // interpolate_kernel (kernels.hpp:133-135), kd = K750 - K500
                        double ck = __dmul_rn(__dadd_rn(__ldg(k5 + j), __dmul_rn(__ldg(kd + j), w)), dts);
                        if (diagonal) ck = __dmul_rn(ck, 0.5);
                        double z = __dmul_rn(__dmul_rn(ck, gai), gbj);
                        const double la = __dmul_rn(gai, xj), lb = __dmul_rn(gbj, xi);
                        if (z > la) z = la;
                        if (z > lb) z = lb;
                        double gsk;
                        if (diagonal) {
                            gsk = __dmul_rn(2.0, __dmul_rn(z, rxi));
                            if (gsk > gai) gsk = gai;
                            ga[i * L] = __dsub_rn(gai, gsk);
                        } else {
                            double gsi = __dmul_rn(z, rxj), gsj = __dmul_rn(z, rxi);
                            if (gsi > gai) gsi = gai;
                            if (gsj > gbj) gsj = gbj;
                            ga[i * L] = __dsub_rn(gai, gsi);
                            gb[j * L] = __dsub_rn(gbj, gsj);
                            gsk = __dadd_rn(gsi, gsj);
                        }
                        const int k = __ldg(glo + j);
                        if (k < 0) { // top rule: the product stays in the last bin
                            gd[(nkr - 1) * L] = __dadd_rn(gd[(nkr - 1) * L], gsk);
                            continue;
                        }
                        const double gk = __dadd_rn(gd[k * L], gsk), gkp = gd[(k + 1) * L];
                        if (gk > 0.0) {
                            const double flux = bott_flux(gsk, gk, gkp, __ldg(cr + j));
                            gd[k * L] = __dsub_rn(gk, flux);
                            gd[(k + 1) * L] = __dadd_rn(gkp, flux);
                        } else {
                            gd[k * L] = gk;
                        }
                    }
                    tr += static_cast<unsigned long long>(nkr - j0);
                }
            }
        }
        if (live) {
            for (int c = 0; c < kNCat; ++c) { // n = g / x
                double *dst = A.bins[c] + static_cast<size_t>(p) * nkr;
                for (int k = 0; k < nkr; ++k) dst[k] = __dmul_rn(G[(c * nkr + k) * L], __ldg(B.rx + k));
            }
            tr_acc += tr;
            pt_acc += 1;
            ev_acc += A.kernel_strategy ? tr : full_evals;
        }
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

} // namespace fsbm
