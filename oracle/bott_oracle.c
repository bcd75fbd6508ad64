/* bott_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker; never shipped).
 *
 * Plain-C restatement of Bott's (1998) flux method for the stochastic collection
 * equation -- A. Bott, "A flux method for the numerical solution of the stochastic
 * collection equation", J. Atmos. Sci. 55, 2284-2293 (1998), Eqs. (2)-(13) and the
 * collision loop of its published coad1d listing -- in the multi-category form WRF's
 * FSBM uses (coal_bott_new -> coll_xxx / coll_xyy / coll_xyz: category a bin i collects
 * category b bin j into category d).  The reference coalbench does NOT implement this
 * scheme ("Kovetz-Olund two-bin splitting chosen over Bott's (1998)
 * flux-form scheme ... a deliberate divergence"), so there is no reference output to pin
 * it to: PARITY UNPINNED against the reference.  It is pinned instead by known-answer
 * tests (tests/test_oracle_bott.py): the SPEC hand examples whose products land in the
 * top bin, a hand-derived flux case, an independent pure-Python restatement, exact
 * positivity, mass conservation to round-off, and the Golovin analytic number decay.
 *
 * What is taken from the reference (so the two schemes share every input): the mass
 * grid, the registry order (accumulation order), the pressure interpolation
 * K = K500 + (K750-K500) w (kernels.hpp:123-135, no FMA), the halved self-pair diagonal
 * and the all_zero pair skip (coalescence.cpp:270-293), the flux-target bin
 * k = GainTable.lo(i,j) and the top rule (m >= x[nkr-1] -> bin nkr-1), and the counters.
 *
 * The scheme, per point and substep (dts = dt / substeps), on MASS per bin g = n x:
 *   for each pair p = (a, b -> d) in registry order with g_a not all zero,
 *     for i, for j (j >= i for self pairs), skipping g_a[i] == 0 or g_b[j] == 0:
 *       ck = K(i,j) dts   (x 1/2 on the self diagonal)
 *       z  = min(ck g_a[i] g_b[j], g_a[i] x_j, g_b[j] x_i)         Bott's x0 with limiters
 *       off-diagonal: gsi = min(z rx_j, g_a[i]), gsj = min(z rx_i, g_b[j])   (rx = 1/x)
 *                     g_a[i] -= gsi;  g_b[j] -= gsj;  gsk = gsi + gsj
 *       self diagonal: gsk = min(2 (z rx_i), g_a[i]);  g_a[i] -= gsk
 *       top (k < 0):  g_d[nkr-1] += gsk
 *       else: gk = g_d[k] + gsk, gkp = g_d[k+1];  if gk > 0:
 *         q = 1/gk, u = (gkp - gk) q, r = gkp q;  x1 = ln(r): log1p(u) for |u| < 1/2,
 *         ln(r + 1e-60) otherwise (Bott's floor), clamped to [ln 1e-60, ln 1e60]
 *         c    = ln(m / x_k) / ln(x_{k+1} / x_k)                        Courant number
 *         flux = x1 == 0 ? gsk c : gsk exp(x1 (1/2 - c)) expm1(x1 c) / x1
 *              = gsk / x1 (exp(x1/2) - exp(x1 (1/2 - c)))               (Bott eq. 13)
 *         flux = min(flux, gsk);  g_d[k] = gk - flux;  g_d[k+1] = gkp + flux
 *   n = g / x at the end.  The updates are Gauss-Seidel (in place, in loop order), as in
 * Bott's listing.  The exp/expm1/log1p form is the cancellation-free restatement of
 * eq. 13 (the two exponentials of eq. 13 cancel when x1 c is small).  Limiters make the
 * scheme positive-definite: no StiffnessError can occur.  Compiled -ffp-contract=off.
 */
#include "coal_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* Courant number of cell (i,j): position of x_i + x_j inside its target bin on the
 * log-mass axis (Bott 1998, eq. 11); 0 for top-rule cells.  Uses the GainTable lo. */
int orc_bott_courant(int nkr, const double *x, const int32_t *g_lo, double *cour) {
    if (nkr < 2) return ORC_DOMAIN;
    for (int i = 0; i < nkr; ++i)
        for (int j = 0; j < nkr; ++j) {
            const size_t e = (size_t)i * nkr + j;
            const int k = g_lo[e];
            if (k < 0) {
                cour[e] = 0.0;
                continue;
            }
            const double m = x[i] + x[j];
            cour[e] = log(m / x[k]) / log(x[k + 1] / x[k]);
        }
    return ORC_OK;
}

static int all_zero(const double *v, int n) {
    for (int k = 0; k < n; ++k)
        if (v[k] != 0.0) return 0;
    return 1;
}

/* Bott's flux of gsk from bin k into bin k+1 (eq. 13, cancellation-free form). */
double orc_bott_flux(double gsk, double gk, double gkp, double c) {
    /* x1 = ln(g_{k+1}/g_k): log1p(u) near 1 (no cancellation), Bott's ln(r + 1e-60) elsewhere,
     * kept inside [ln 1e-60, ln 1e60] (Bott's floor mirrored above) so no term overflows */
    const double q = 1.0 / gk, u = (gkp - gk) * q, r = gkp * q;
    const double lo = -138.15510557964274; /* ln(1e-60), Bott's g_min */
    double x1 = (u > -0.5 && u < 0.5) ? log1p(u) : log(r + 1e-60);
    if (x1 < lo) x1 = lo;
    if (x1 > -lo) x1 = -lo;
    double flux;
    if (x1 == 0.0) flux = gsk * c;
    else flux = gsk * exp(x1 * (0.5 - c)) * expm1(x1 * c) / x1;
    return flux < gsk ? flux : gsk;
}

int orc_bott_step(int nkr, const double *x, int npairs, const int *abd, const double *t750,
                  const double *t500, const int32_t *g_lo, const double *cour,
                  double *const bins[ORC_NCAT], double pressure, double dt, int substeps,
                  int kernel_strategy, uint64_t *counters) {
    if (!(dt > 0.0)) return ORC_DOMAIN;
    if (substeps < 1) return ORC_DOMAIN;
    double *g = (double *)malloc(sizeof(double) * (ORC_NCAT + 1) * nkr);
    double *rx = g + ORC_NCAT * nkr; /* 1 / x */
    for (int k = 0; k < nkr; ++k) rx[k] = 1.0 / x[k];
    const double w = orc_pressure_weight(pressure);
    const double dts = dt / substeps;
    uint64_t triples = 0;
    for (int c = 0; c < ORC_NCAT; ++c)
        for (int k = 0; k < nkr; ++k) g[c * nkr + k] = bins[c][k] * x[k];
    for (int step = 0; step < substeps; ++step) {
        for (int p = 0; p < npairs; ++p) {
            const int a = abd[3 * p], b = abd[3 * p + 1], d = abd[3 * p + 2];
            double *ga = g + a * nkr, *gb = g + b * nkr, *gd = g + d * nkr;
            const int self = a == b;
            if (all_zero(ga, nkr)) continue; /* coalescence.cpp:270-273 */
            for (int i = 0; i < nkr; ++i) {
                const int j0 = self ? i : 0;
                const size_t row = ((size_t)p * nkr + i) * nkr;
                for (int j = j0; j < nkr; ++j) {
                    const double gai = ga[i], gbj = gb[j];
                    if (gai == 0.0 || gbj == 0.0) continue;
                    const int diagonal = self && i == j;
                    double ck = orc_interpolate(t750[row + j], t500[row + j], w) * dts;
                    if (diagonal) ck *= 0.5;
                    double z = ck * gai * gbj;
                    const double la = gai * x[j], lb = gbj * x[i];
                    if (z > la) z = la;
                    if (z > lb) z = lb;
                    double gsk;
                    if (diagonal) {
                        gsk = 2.0 * (z * rx[i]);
                        if (gsk > gai) gsk = gai;
                        ga[i] = gai - gsk;
                    } else {
                        double gsi = z * rx[j], gsj = z * rx[i];
                        if (gsi > gai) gsi = gai;
                        if (gsj > gbj) gsj = gbj;
                        ga[i] = gai - gsi;
                        gb[j] = gb[j] - gsj;
                        gsk = gsi + gsj;
                    }
                    const size_t e = (size_t)i * nkr + j;
                    const int k = g_lo[e];
                    if (k < 0) {
                        gd[nkr - 1] += gsk;
                        continue;
                    }
                    const double gk = gd[k] + gsk, gkp = gd[k + 1];
                    if (gk > 0.0) {
                        const double flux = orc_bott_flux(gsk, gk, gkp, cour[e]);
                        gd[k] = gk - flux;
                        gd[k + 1] = gkp + flux;
                    } else {
                        gd[k] = gk;
                    }
                }
                triples += (uint64_t)(nkr - j0);
            }
        }
    }
    for (int c = 0; c < ORC_NCAT; ++c)
        for (int k = 0; k < nkr; ++k) bins[c][k] = g[c * nkr + k] * rx[k];
    free(g);
    if (counters) {
        counters[0] += triples;
        counters[1] += 1;
        counters[2] += kernel_strategy ? triples : (uint64_t)npairs * nkr * nkr; /* once per call */
    }
    return ORC_OK;
}

/* orc_bott_step over every mask-true point of a whole (i,k,j) domain (bins category-major
 * [6][np*nkr], point p = (i*nk + k)*nj + j), split over nthreads contiguous point ranges
 * (the scheme is per point, so the split does not change any value). */

typedef struct {
    int nkr, npairs, substeps, kstrat;
    const double *x, *t750, *t500, *cour, *pressure;
    const int *abd;
    const int32_t *g_lo;
    const uint8_t *mask;
    double *bins, dt;
    size_t np, begin, end;
    uint64_t counters[3];
} bott_chunk;

static void *bott_worker(void *arg) {
    bott_chunk *g = (bott_chunk *)arg;
    for (size_t p = g->begin; p < g->end; ++p) {
        if (g->mask && !g->mask[p]) continue;
        double *b6[ORC_NCAT];
        for (int c = 0; c < ORC_NCAT; ++c) b6[c] = g->bins + ((size_t)c * g->np + p) * g->nkr;
        orc_bott_step(g->nkr, g->x, g->npairs, g->abd, g->t750, g->t500, g->g_lo, g->cour, b6,
                      g->pressure[p], g->dt, g->substeps, g->kstrat, g->counters);
    }
    return NULL;
}

int orc_bott_step_grid(size_t np, int nkr, const double *x, int npairs, const int *abd,
                       const double *t750, const double *t500, const int32_t *g_lo,
                       const double *cour, const uint8_t *mask, const double *pressure,
                       double *bins, double dt, int substeps, int kernel_strategy, int nthreads,
                       uint64_t *counters) {
    if (!(dt > 0.0) || substeps < 1) return ORC_DOMAIN;
    if (nthreads < 1) nthreads = 1;
    bott_chunk *ch = (bott_chunk *)calloc((size_t)nthreads, sizeof(bott_chunk));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int w = 0; w < nthreads; ++w) {
        bott_chunk *g = &ch[w];
        g->nkr = nkr; g->npairs = npairs; g->substeps = substeps; g->kstrat = kernel_strategy;
        g->x = x; g->t750 = t750; g->t500 = t500; g->cour = cour; g->pressure = pressure;
        g->abd = abd; g->g_lo = g_lo; g->mask = mask; g->bins = bins; g->dt = dt; g->np = np;
        g->begin = np * (size_t)w / (size_t)nthreads;
        g->end = np * (size_t)(w + 1) / (size_t)nthreads;
        if (nthreads > 1) pthread_create(&th[w], NULL, bott_worker, g);
        else bott_worker(g);
    }
    for (int w = 0; w < nthreads; ++w) {
        if (nthreads > 1) pthread_join(th[w], NULL);
        if (counters)
            for (int k = 0; k < 3; ++k) counters[k] += ch[w].counters[k];
    }
    free(ch);
    free(th);
    return ORC_OK;
}
