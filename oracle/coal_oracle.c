/* coal_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker; never shipped).
 *
 * Plain-C restatement of the reference coalbench hot path.  Compiled with
 * -ffp-contract=off, as the reference is (proj/CMakeLists.txt:12-15), so every
 * product/sum rounds exactly where the reference's does.  Each function cites
 * the reference file:line it restates.  Pinned bit-for-bit against the
 * reference library itself (oracle/_ref) by tests/test_oracle.py.
 */
#define _GNU_SOURCE
#include "coal_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- L0: mass grid (proj/src/mass_grid.cpp:10-25) ---------------------- */
int orc_mass_grid(int nkr, double x1, double ratio, double *x) {
    if (nkr < 2) return ORC_DOMAIN;
    if (!(x1 > 0.0) || !isfinite(x1)) return ORC_DOMAIN;
    if (!(ratio > 1.0) || !isfinite(ratio)) return ORC_DOMAIN;
    x[0] = x1;
    for (int k = 1; k < nkr; ++k) x[k] = x[k - 1] * ratio; /* repeated multiply, not pow */
    return ORC_OK;
}

/* proj/src/mass_grid.cpp:27-48 */
int orc_exponential_init(int nkr, const double *x, double n_total, double xbar, double *out) {
    if (!(n_total >= 0.0) || !isfinite(n_total)) return ORC_DOMAIN;
    if (!(xbar > 0.0) || !isfinite(xbar)) return ORC_DOMAIN;
    for (int k = 0; k < nkr; ++k) out[k] = 0.0;
    if (n_total == 0.0) return ORC_OK;
    double wsum = 0.0;
    for (int k = 0; k < nkr; ++k) {
        out[k] = x[k] * exp(-x[k] / xbar);
        wsum += out[k];
    }
    if (wsum == 0.0) return ORC_DOMAIN;
    for (int k = 0; k < nkr; ++k) out[k] = n_total * (out[k] / wsum);
    return ORC_OK;
}

/* ---- gain table (proj/src/coalescence.cpp:36-67) ----------------------- */
int orc_gain_table(int nkr, const double *x, double ratio, int32_t *lo, double *w_lo,
                   double *w_hi, double *top) {
    if (nkr < 2) return ORC_DOMAIN;
    const double xt = x[nkr - 1];
    const double inv_log_ratio = 1.0 / log(ratio);
    const double log_x0 = log(x[0]);
    for (int i = 0; i < nkr; ++i)
        for (int j = 0; j < nkr; ++j) {
            const size_t e = (size_t)i * nkr + j;
            const double m = x[i] + x[j];
            lo[e] = 0;
            w_lo[e] = 0.0;
            w_hi[e] = 0.0;
            top[e] = 0.0;
            if (m >= xt) { /* top-bin rule: mass-conserving */
                lo[e] = -1;
                top[e] = m / xt;
                continue;
            }
            int k = (int)floor((log(m) - log_x0) * inv_log_ratio);
            if (k < 0) k = 0;
            if (k > nkr - 2) k = nkr - 2;
            while (k + 1 < nkr - 1 && x[k + 1] <= m) ++k;
            while (k > 0 && x[k] > m) --k;
            lo[e] = k;
            const double width = x[k + 1] - x[k];
            w_lo[e] = (x[k + 1] - m) / width;
            w_hi[e] = (m - x[k]) / width;
        }
    return ORC_OK;
}

/* ---- kernels (proj/src/kernels.cpp) ------------------------------------ */
/* Category order: liquid, ice1, ice2, ice3, snow, graupel (kernels.hpp:17-26) */
enum { L_ = 0, I1 = 1, I2 = 2, I3 = 3, S_ = 4, G_ = 5 };

int orc_default_registry(int *abd) { /* kernels.cpp:65-93 */
    static const int r[20][3] = {
        {L_, L_, L_}, {I1, I1, I1}, {I2, I2, I2}, {I3, I3, I3}, {S_, S_, S_},
        {G_, G_, G_}, {L_, I1, I1}, {L_, I2, I2}, {L_, I3, I3}, {L_, S_, S_},
        {L_, G_, G_}, {I1, S_, S_}, {I2, S_, S_}, {I3, S_, S_}, {I1, G_, G_},
        {I2, G_, G_}, {I3, G_, G_}, {S_, G_, G_}, {S_, L_, G_}, {G_, L_, G_},
    };
    for (int p = 0; p < 20; ++p)
        for (int q = 0; q < 3; ++q) abd[3 * p + q] = r[p][q];
    return 20;
}

static double family_value(int family, double coeff, double xi, double xj) { /* kernels.cpp:16-34 */
    switch (family) {
    case 0: return coeff;
    case 1: return coeff * (xi + xj);
    case 2: return coeff * xi * xj;
    case 3: {
        double ri = cbrt(xi), rj = cbrt(xj);
        double sigma = (ri + rj) * (ri + rj);
        return coeff * sigma * sqrt(ri * ri + rj * rj);
    }
    }
    return NAN;
}

int orc_build_tables(int nkr, const double *x, int npairs, int family, double coeff,
                     double level_scale, double pair_scale_step, double *t750, double *t500) {
    if (!(coeff >= 0.0) || !isfinite(coeff)) return ORC_DOMAIN;
    if (!(level_scale >= 0.0) || !isfinite(level_scale)) return ORC_DOMAIN;
    if (!(pair_scale_step >= 0.0) || !isfinite(pair_scale_step)) return ORC_DOMAIN;
    if (family < 0 || family > 3) return ORC_DOMAIN;
    for (int p = 0; p < npairs; ++p) {
        const double pair_scale = 1.0 + pair_scale_step * p;
        for (int i = 0; i < nkr; ++i)
            for (int j = 0; j < nkr; ++j) {
                const size_t idx = ((size_t)p * nkr + i) * nkr + j;
                double v = family_value(family, coeff, x[i], x[j]) * pair_scale;
                t750[idx] = v;
                t500[idx] = v * level_scale;
            }
    }
    return ORC_OK;
}

double orc_pressure_weight(double pressure) { /* kernels.hpp:123-129 */
    double w = (pressure - 500.0) / (750.0 - 500.0);
    if (w < 0.0) w = 0.0;
    if (w > 1.0) w = 1.0;
    return w;
}

double orc_interpolate(double k750, double k500, double w) { /* kernels.hpp:133-135 */
    return k500 + (k750 - k500) * w;
}

/* ---- coal_step (proj/src/coalescence.cpp:204-339) ----------------------- */
static int all_zero(const double *v, int n) { /* coalescence.cpp:195-200 */
    for (int k = 0; k < n; ++k)
        if (v[k] != 0.0) return 0;
    return 1;
}

int orc_coal_step(int nkr, const double *x, int npairs, const int *abd, const double *t750,
                  const double *t500, const int32_t *g_lo, const double *g_wlo,
                  const double *g_whi, const double *g_top, double *const bins[ORC_NCAT],
                  double pressure, double dt, int substeps, int kernel_strategy,
                  uint64_t *counters, int *err_cat, int *err_bin) {
    (void)x;
    if (!(dt > 0.0)) return ORC_DOMAIN;
    if (substeps < 1) return ORC_DOMAIN;
    const int on_demand = kernel_strategy != 0;
    double *work = (double *)malloc(sizeof(double) * 2 * ORC_NCAT * nkr);
    double *delta = work + ORC_NCAT * nkr;
    double *pk = NULL;
    const double w = orc_pressure_weight(pressure);
    if (!on_demand) { /* precompute_all, kernels.cpp:154-172 */
        pk = (double *)malloc(sizeof(double) * (size_t)npairs * nkr * nkr);
        size_t idx = 0;
        for (int p = 0; p < npairs; ++p)
            for (int i = 0; i < nkr; ++i)
                for (int j = 0; j < nkr; ++j, ++idx)
                    pk[idx] = orc_interpolate(t750[idx], t500[idx], w);
    }
    const double dt_sub = dt / substeps;
    uint64_t triples = 0;
    int st = ORC_OK;
    for (int step = 0; step < substeps && st == ORC_OK; ++step) {
        for (int c = 0; c < ORC_NCAT; ++c) {
            memcpy(work + c * nkr, bins[c], sizeof(double) * nkr);
            memset(delta + c * nkr, 0, sizeof(double) * nkr);
        }
        for (int p = 0; p < npairs; ++p) {
            const int a = abd[3 * p], b = abd[3 * p + 1], d = abd[3 * p + 2];
            const double *na = work + a * nkr, *nb = work + b * nkr;
            double *da = delta + a * nkr, *db = delta + b * nkr, *dd = delta + d * nkr;
            const int self = a == b;
            if (all_zero(na, nkr)) continue;
            for (int i = 0; i < nkr; ++i) {
                const int j0 = self ? i : 0;
                const double nai = na[i];
                const size_t row = ((size_t)p * nkr + i) * nkr;
                for (int j = j0; j < nkr; ++j) {
                    const double kij = on_demand ? orc_interpolate(t750[row + j], t500[row + j], w)
                                                 : pk[row + j];
                    double rate = kij * nai * nb[j];
                    if (rate == 0.0) continue;
                    const int diagonal = self && i == j;
                    if (diagonal) rate *= 0.5;
                    const double dn = rate * dt_sub;
                    if (diagonal) {
                        da[i] -= 2.0 * dn;
                    } else {
                        da[i] -= dn;
                        db[j] -= dn;
                    }
                    const size_t e = (size_t)i * nkr + j;
                    if (g_lo[e] >= 0) {
                        dd[g_lo[e]] += dn * g_wlo[e];
                        dd[g_lo[e] + 1] += dn * g_whi[e];
                    } else {
                        dd[nkr - 1] += dn * g_top[e];
                    }
                }
                triples += (uint64_t)(nkr - j0);
            }
        }
        /* Jacobi apply + stiffness (coalescence.cpp:313-328) */
        for (int c = 0; c < ORC_NCAT && st == ORC_OK; ++c)
            for (int k = 0; k < nkr; ++k) {
                const double v = work[c * nkr + k] + delta[c * nkr + k];
                if (v < 0.0) {
                    if (err_cat) *err_cat = c;
                    if (err_bin) *err_bin = k;
                    st = ORC_STIFF;
                    break;
                }
                bins[c][k] = v;
            }
    }
    free(work);
    free(pk);
    if (st == ORC_STIFF) return st; /* the reference throws before counting */
    if (counters) {
        counters[0] += triples;
        counters[1] += 1;
        counters[2] += on_demand ? triples : (uint64_t)npairs * nkr * nkr;
    }
    return ORC_OK;
}

/* ---- rng (proj/include/coalbench/rng.hpp:10-32) ------------------------ */
uint64_t orc_splitmix_next(uint64_t *s) {
    uint64_t z = (*s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
double orc_uniform01(uint64_t *s) { return (double)(orc_splitmix_next(s) >> 11) * 0x1.0p-53; }
uint64_t orc_bounded(uint64_t *s, uint64_t bound) {
    return (uint64_t)(((unsigned __int128)orc_splitmix_next(s) * bound) >> 64);
}

/* ---- synthetic case (proj/src/driver.cpp:223-285) ----------------------- */
int orc_synthetic_case(int ni, int nk, int nj, double cloud_fraction, uint64_t seed, int nkr,
                       double x1, double ratio, double number_density, double *temperature,
                       double *pressure, double *bins) {
    if (ni < 1 || nk < 1 || nj < 1) return ORC_DOMAIN;
    if (!(cloud_fraction >= 0.0 && cloud_fraction <= 1.0)) return ORC_DOMAIN;
    if (!(number_density >= 0.0) || !isfinite(number_density)) return ORC_DOMAIN;
    double *x = (double *)malloc(sizeof(double) * nkr);
    int st = orc_mass_grid(nkr, x1, ratio, x);
    if (st) { free(x); return st; }
    const size_t np = (size_t)ni * nk * nj;
    if (bins) memset(bins, 0, sizeof(double) * ORC_NCAT * np * nkr); /* NULL: T/P only */
    const size_t n_cloudy = (size_t)llround(cloud_fraction * (double)np);
    uint64_t rng = seed;
    uint32_t *perm = (uint32_t *)malloc(sizeof(uint32_t) * np);
    uint8_t *cloudy = (uint8_t *)calloc(np, 1);
    for (size_t p = 0; p < np; ++p) perm[p] = (uint32_t)p;
    for (size_t p = np - 1; p > 0; --p) {
        size_t q = (size_t)orc_bounded(&rng, p + 1);
        uint32_t t = perm[p]; perm[p] = perm[q]; perm[q] = t;
    }
    for (size_t c = 0; c < n_cloudy; ++c) cloudy[perm[c]] = 1;
    for (size_t p = 0; p < np; ++p) {
        if (cloudy[p]) temperature[p] = 240.0 + 60.0 * orc_uniform01(&rng);
        else temperature[p] = (orc_splitmix_next(&rng) & 1) ? 210.0 : 180.0;
    }
    for (int i = 0; i < ni; ++i)
        for (int k = 0; k < nk; ++k)
            for (int j = 0; j < nj; ++j) {
                const double frac = nk > 1 ? (double)k / (nk - 1) : 0.0;
                pressure[((size_t)i * nk + k) * nj + j] = 900.0 + (400.0 - 900.0) * frac;
            }
    const int kbar = nkr - 1 < nkr / 3 ? nkr - 1 : nkr / 3;
    const double xbar = x[kbar];
    for (size_t p = 0; bins && p < np && st == ORC_OK; ++p) {
        if (!cloudy[p]) continue;
        const double n_total = number_density * (0.5 + orc_uniform01(&rng));
        st = orc_exponential_init(nkr, x, n_total, xbar, bins + p * nkr); /* liquid = 0 */
    }
    free(perm);
    free(cloudy);
    free(x);
    return st;
}

int orc_thunderstorm_point(int nkr, const double *x, uint64_t seed, uint64_t p, double *out) {
    static const double s[ORC_NCAT] = {1.0, 0.25, 0.25, 0.25, 0.25, 0.25};
    uint64_t rng = seed ^ p;
    for (int c = 0; c < ORC_NCAT; ++c) {
        const double u = orc_uniform01(&rng);
        int kb = nkr / 3 + c * nkr / 16;
        if (kb > nkr - 1) kb = nkr - 1;
        int st = orc_exponential_init(nkr, x, 1e6 * (0.5 + u) * s[c], x[kb], out + c * nkr);
        if (st) return st;
    }
    return ORC_OK;
}

int orc_thunderstorm_block(int nkr, const double *x, uint64_t seed, uint64_t p0, uint64_t n,
                           const uint8_t *mask, double *bins) {
    double *tmp = (double *)malloc(sizeof(double) * ORC_NCAT * nkr);
    for (uint64_t q = 0; q < n; ++q) {
        const int on = mask ? mask[q] != 0 : 1;
        if (on && orc_thunderstorm_point(nkr, x, seed, p0 + q, tmp)) { free(tmp); return ORC_DOMAIN; }
        for (int c = 0; c < ORC_NCAT; ++c)
            for (int k = 0; k < nkr; ++k)
                bins[(size_t)c * n * nkr + q * nkr + k] = on ? tmp[c * nkr + k] : 0.0;
    }
    free(tmp);
    return ORC_OK;
}

uint64_t orc_fission_predicates(uint64_t npoints, const double *temperature, uint8_t *mask) {
    uint64_t count = 0; /* driver.cpp:198-211 */
    for (uint64_t p = 0; p < npoints; ++p) {
        const double t = temperature[p];
        const int on = t > 193.15 && t > 223.15;
        mask[p] = (uint8_t)on;
        count += (uint64_t)on;
    }
    return count;
}

/* ---- grid driver, phase 2 (proj/src/driver.cpp:384-430) ----------------- */
typedef struct {
    int ni, nk, nj, nkr, npairs, substeps, kstrat;
    const double *x, *t750, *t500, *g_wlo, *g_whi, *g_top, *pressure;
    const int32_t *g_lo;
    const int *abd;
    const uint8_t *mask;
    double *bins, dt;
    size_t begin, end;
    uint64_t counters[3];
    int st, err5[5];
} grid_chunk;

static void *grid_worker(void *arg) {
    grid_chunk *g = (grid_chunk *)arg;
    const size_t np = (size_t)g->ni * g->nk * g->nj;
    const size_t inner = (size_t)g->nk * g->ni;
    for (size_t u = g->begin; u < g->end && g->st == ORC_OK; ++u) {
        const int j = (int)(u / inner);
        const size_t rem = u % inner;
        const int k = (int)(rem / g->ni);
        const int i = (int)(rem % g->ni);
        const size_t p = ((size_t)i * g->nk + k) * g->nj + j;
        if (!g->mask[p]) continue;
        double *b6[ORC_NCAT];
        for (int c = 0; c < ORC_NCAT; ++c) b6[c] = g->bins + (size_t)c * np * g->nkr + p * g->nkr;
        int ec = -1, eb = -1;
        int st = orc_coal_step(g->nkr, g->x, g->npairs, g->abd, g->t750, g->t500, g->g_lo,
                               g->g_wlo, g->g_whi, g->g_top, b6, g->pressure[p], g->dt,
                               g->substeps, g->kstrat, g->counters, &ec, &eb);
        if (st != ORC_OK) {
            g->st = st;
            g->err5[0] = ec; g->err5[1] = eb;
            g->err5[2] = i + 1; g->err5[3] = k + 1; g->err5[4] = j + 1;
        }
    }
    return NULL;
}

int orc_step_grid(int ni, int nk, int nj, int nkr, const double *x, int npairs, const int *abd,
                  const double *t750, const double *t500, const int32_t *g_lo,
                  const double *g_wlo, const double *g_whi, const double *g_top,
                  const uint8_t *mask, const double *pressure, double *bins, double dt,
                  int substeps, int kernel_strategy, int nthreads, uint64_t *counters,
                  int *err5) {
    const size_t total = (size_t)ni * nk * nj;
    if (nthreads < 1) nthreads = 1;
    grid_chunk *ch = (grid_chunk *)calloc((size_t)nthreads, sizeof(grid_chunk));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int w = 0; w < nthreads; ++w) {
        grid_chunk *g = &ch[w];
        g->ni = ni; g->nk = nk; g->nj = nj; g->nkr = nkr; g->npairs = npairs;
        g->substeps = substeps; g->kstrat = kernel_strategy;
        g->x = x; g->t750 = t750; g->t500 = t500; g->g_lo = g_lo; g->g_wlo = g_wlo;
        g->g_whi = g_whi; g->g_top = g_top; g->pressure = pressure; g->abd = abd;
        g->mask = mask; g->bins = bins; g->dt = dt;
        g->begin = total * (size_t)w / (size_t)nthreads;
        g->end = total * (size_t)(w + 1) / (size_t)nthreads;
        if (nthreads > 1) pthread_create(&th[w], NULL, grid_worker, g);
        else grid_worker(g);
    }
    if (nthreads > 1)
        for (int w = 0; w < nthreads; ++w) pthread_join(th[w], NULL);
    int st = ORC_OK;
    for (int w = 0; w < nthreads; ++w) {
        if (counters)
            for (int q = 0; q < 3; ++q) counters[q] += ch[w].counters[q];
        if (st == ORC_OK && ch[w].st != ORC_OK) { /* lowest worker wins (driver.cpp:79-83) */
            st = ch[w].st;
            if (err5) memcpy(err5, ch[w].err5, sizeof(int) * 5);
        }
    }
    free(ch);
    free(th);
    return st;
}
