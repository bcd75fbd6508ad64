// coal_exact.cuh -- FSBM_NUMERICS_EXACT: bitwise-identical coal_step on device.
//
// One thread = one mask-true grid point, executing coal_step
// (proj/src/coalescence.cpp:204-339) in the reference's exact operation order:
// pairs in registry order, i outer, j inner (j >= i for self pairs), every
// product/sum rounded separately (__dmul_rn/__dadd_rn: no FMA contraction, as
// the reference's -ffp-contract=off, proj/CMakeLists.txt:12-15).  Per-point
// working/delta arrays live in a per-warp global "arena" laid out
// [array][bin][lane] so that the 32 lanes of a warp (32 points walking the
// same (pair,i,j) in lockstep) touch one contiguous 256-byte line per access,
// while the kernel tables and gain entries are warp-uniform broadcast loads.
// This is the device analogue of the reference's collapse-3 + arena variant
// (driver.cpp:402-414, coalescence.cpp:82-187).  It is the bit-exact mode;
// the throughput path is coal_fast.cuh.
#pragma once

#include "fsbm_common.cuh"

namespace fsbm {

constexpr int kExactThreads = 128;

__device__ inline void flush_counters(const StepArgs &A, unsigned long long tr,
                                      unsigned long long pts, unsigned long long ev) {
    for (int o = 16; o > 0; o >>= 1) {
        tr += __shfl_down_sync(0xffffffffu, tr, o);
        pts += __shfl_down_sync(0xffffffffu, pts, o);
        ev += __shfl_down_sync(0xffffffffu, ev, o);
    }
    if ((threadIdx.x & 31) == 0 && (tr | pts | ev)) {
        atomicAdd(&A.counters[0], tr);
        atomicAdd(&A.counters[1], pts);
        atomicAdd(&A.counters[2], ev);
    }
}

/// da[i] is held in a register across the j loop (its updates, and the gains that land on the
/// same element, are applied in the reference's order).  (Deltas in shared memory -- 4 warps
/// per SM -- measured 4x slower: the arena's 32 warps per SM hide its L2 latency.)
__global__ void __launch_bounds__(kExactThreads, 8) coal_exact_kernel(StepArgs A, double *arena) {
    if (A.stale && *A.stale) return; // stale mask: the step must not touch the state
    const int nkr = A.nkr;
    const uint32_t nact = *A.nactive;
    const int lane = threadIdx.x & 31;
    const size_t gwarp = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    constexpr int L = 32; // lane stride inside the arena
    const size_t span = static_cast<size_t>(kNCat) * nkr * L;
    double *W = arena + gwarp * 2 * span + lane;
    double *Dl = W + span;
    const int npairs = A.pairs.npairs;
    const unsigned long long full_evals = static_cast<unsigned long long>(npairs) * nkr * nkr;

    unsigned long long tr_acc = 0, pt_acc = 0, ev_acc = 0;
    // Grid-stride over whole warps so every lane of a warp stays in the loop.
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < nact; base += stride) {
        const uint32_t idx = base + lane;
        const bool live = idx < nact;
        const uint32_t p = live ? A.active[idx] : 0u;
        const double w = live ? pressure_weight(A.pressure[p]) : 0.0;
        bool failed = !live;
        unsigned long long tr = 0;
        for (int s = 0; s < A.substeps && !failed; ++s) {
            // working copies + zeroed deltas (coalescence.cpp:256-259)
            for (int c = 0; c < kNCat; ++c) {
                const double *src = A.bins[c] + static_cast<size_t>(p) * nkr;
                for (int k = 0; k < nkr; ++k) {
                    W[(c * nkr + k) * L] = src[k];
                    Dl[(c * nkr + k) * L] = 0.0;
                }
            }
            for (int q = 0; q < npairs; ++q) {
                const int a = A.pairs.a[q], b = A.pairs.b[q], d = A.pairs.d[q];
                const bool self = a == b;
                // the working copies are read-only during the pass loop (only the deltas are
                // written): restrict lets their loads run ahead of the delta stores
                const double *__restrict__ na = W + a * nkr * L;
                const double *__restrict__ nb = W + b * nkr * L;
                double *da = Dl + a * nkr * L;
                double *db = Dl + b * nkr * L;
                double *dd = Dl + d * nkr * L;
                bool any = false; // all_zero (coalescence.cpp:195-200,270-273)
                for (int k = 0; k < nkr && !any; ++k) any = na[k * L] != 0.0;
                if (!any) continue;
                for (int i = 0; i < nkr; ++i) {
                    const int j0 = self ? i : 0;
                    const double nai = na[i * L];
                    const double *k5 = A.k500 + (static_cast<size_t>(q) * nkr + i) * nkr;
                    const double *kd = A.kd + (static_cast<size_t>(q) * nkr + i) * nkr;
                    const int32_t *glo = A.g_lo + static_cast<size_t>(i) * nkr;
                    const double *gwl = A.g_wlo + static_cast<size_t>(i) * nkr;
                    const double *gwh = A.g_whi + static_cast<size_t>(i) * nkr;
                    const double *gtp = A.g_top + static_cast<size_t>(i) * nkr;
                    // da[i] in a register for the row: db[j] never aliases it (a != b, or the
                    // self diagonal, which updates da[i] itself); a gain landing on (a, i) is
                    // folded into the register in its place in the update sequence
                    double dai = da[i * L];
                    const bool dsa = d == a;
#pragma unroll 4
                    for (int j = j0; j < nkr; ++j) {
                        // interpolate_kernel: K500 + (K750-K500)*w (kernels.hpp:133-135);
                        // kd holds the (K750-K500) difference, bit-identical.
                        const double kij = __dadd_rn(__ldg(k5 + j), __dmul_rn(__ldg(kd + j), w));
                        double rate = __dmul_rn(__dmul_rn(kij, nai), nb[j * L]);
                        if (rate == 0.0) continue;
                        const bool diagonal = self && i == j;
                        if (diagonal) rate = __dmul_rn(rate, 0.5);
                        const double dn = __dmul_rn(rate, A.dt_sub);
                        if (diagonal) {
                            dai = __dsub_rn(dai, __dmul_rn(2.0, dn));
                        } else {
                            dai = __dsub_rn(dai, dn);
                            db[j * L] = __dsub_rn(db[j * L], dn);
                        }
                        const int lo = __ldg(glo + j);
                        if (lo >= 0) {
                            const double v0 = __dmul_rn(dn, __ldg(gwl + j)), v1 = __dmul_rn(dn, __ldg(gwh + j));
                            if (dsa && lo == i) dai = __dadd_rn(dai, v0);
                            else dd[lo * L] = __dadd_rn(dd[lo * L], v0);
                            if (dsa && lo + 1 == i) dai = __dadd_rn(dai, v1);
                            else dd[(lo + 1) * L] = __dadd_rn(dd[(lo + 1) * L], v1);
                        } else {
                            const double v = __dmul_rn(dn, __ldg(gtp + j));
                            if (dsa && nkr - 1 == i) dai = __dadd_rn(dai, v);
                            else dd[(nkr - 1) * L] = __dadd_rn(dd[(nkr - 1) * L], v);
                        }
                    }
                    da[i * L] = dai;
                    tr += static_cast<unsigned long long>(nkr - j0);
                }
            }
            // Jacobi apply + stiffness check (coalescence.cpp:313-328)
            for (int c = 0; c < kNCat && !failed; ++c) {
                double *out = A.bins[c] + static_cast<size_t>(p) * nkr;
                for (int k = 0; k < nkr; ++k) {
                    const double v = __dadd_rn(W[(c * nkr + k) * L], Dl[(c * nkr + k) * L]);
                    if (v < 0.0) {
                        report_stiffness(A, p, c, k, v);
                        failed = true;
                        break;
                    }
                    out[k] = v;
                }
            }
        }
        if (!failed) {
            tr_acc += tr;
            pt_acc += 1;
            ev_acc += A.kernel_strategy ? tr : full_evals;
        }
    }
    flush_counters(A, tr_acc, pt_acc, ev_acc);
}

} // namespace fsbm
