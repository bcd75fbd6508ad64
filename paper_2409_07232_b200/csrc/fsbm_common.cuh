// fsbm_common.cuh -- device-side shared definitions for the FSBM coalescence kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fsbm {

constexpr int kNCat = 6;
constexpr int kMaxPairs = 64;

// Interpolation reference levels (kernels.hpp:83-84) and gates (driver.hpp:17-20).
constexpr double kLowPressure = 500.0;
constexpr double kHighPressure = 750.0;
constexpr double kOuterGateK = 193.15;
constexpr double kCoalGateK = 223.15;

/// pressure_weight (kernels.hpp:123-129), same operation order.
__host__ __device__ inline double pressure_weight(double p) {
    double w = (p - kLowPressure) / (kHighPressure - kLowPressure);
    if (w < 0.0) w = 0.0;
    if (w > 1.0) w = 1.0;
    return w;
}

/// Registry + per-pair flags, passed by value to kernels.
struct PairTable {
    int npairs;
    int8_t a[kMaxPairs], b[kMaxPairs], d[kMaxPairs];
};

/// Everything a step kernel needs besides the state.
struct StepArgs {
    int nkr;
    int ni, nk, nj;            // extents of this launch's slab (points p are slab-local)
    int ids, kds, jds;         // domain origin (1-based)
    int i_off;                 // global i offset of the slab (host path processes i-chunks)
    int ni_glob;               // global ni (serial-order keys are domain-global)
    const unsigned long long *stale; // non-zero: stale mask detected -> do nothing
    double dt_sub;
    int substeps;
    int kernel_strategy;       // 0 precomputed / 1 on_demand (counters only)
    uint32_t nactive_host;     // upper bound used for grid sizing (may be > real)
    const uint32_t *active;    // compacted mask-true point indices
    const uint32_t *nactive;   // device count
    double *bins[kNCat];
    const double *pressure;
    // tables: k500 and kd = k750 - k500, layout [pair][i][j] (kernels.hpp:105-107)
    const double *k500, *kd;
    const int32_t *g_lo;       // GainTable (coalescence.cpp:36-67), [i][j]
    const double *g_wlo, *g_whi, *g_top;
    // error / counter sink
    unsigned long long *err_key;   // min over failing points of (order<<20 | c*nkr+bin)
    unsigned long long *err_aux;   // {bits of the winning point's negative value, lock}
    unsigned long long *counters;  // {triples, points, kernel_evals}
    const int4 *tiles;             // (its, ite, jts, jte) 1-based, or null
    int ntiles;
    PairTable pairs;
};

/// Serial-order key of point p for StiffnessError reporting: (tile, j, k, i).
__device__ inline unsigned long long order_key(const StepArgs &A, uint32_t p) {
    const uint32_t j = p % A.nj;
    const uint32_t k = (p / A.nj) % A.nk;
    const uint32_t i = p / (A.nj * A.nk) + A.i_off; // global (0-based) i
    unsigned long long t = 0;
    if (A.tiles) {
        for (int q = 0; q < A.ntiles; ++q) {
            const int4 T = A.tiles[q];
            const int gi = (int)i + A.ids, gj = (int)j + A.jds;
            if (gi >= T.x && gi <= T.y && gj >= T.z && gj <= T.w) { t = q; break; }
        }
    }
    const unsigned long long np = (unsigned long long)A.ni_glob * A.nk * A.nj;
    return t * np + ((unsigned long long)j * A.nk + k) * A.ni_glob + i;
}

/// Records (key, value) if key is the smallest so far.  The value rides with the key
/// (the reference's message prints it, coalescence.cpp:319-325), so the pair is updated
/// under a tiny spin lock: this is the error path only, a failing step takes it a
/// handful of times.
__device__ inline void report_stiffness(const StepArgs &A, uint32_t p, int c, int bin, double v) {
    const unsigned long long key = (order_key(A, p) << 20) | (unsigned long long)(c * A.nkr + bin);
    volatile unsigned long long *vk = A.err_key;
    if (key >= *vk) return;
    while (atomicCAS(A.err_aux + 1, 0ull, 1ull) != 0ull) __nanosleep(64);
    __threadfence();
    if (key < *vk) {
        *vk = key;
        *reinterpret_cast<volatile unsigned long long *>(A.err_aux) =
            static_cast<unsigned long long>(__double_as_longlong(v));
    }
    __threadfence();
    atomicExch(A.err_aux + 1, 0ull);
}

} // namespace fsbm
