/* coal_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's FSBM collision-coalescence hot path
 * (coalbench, /root/reference/proj).  Used exclusively as the parity checker by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.  The product
 * (paper_2409_07232_b200/) never links or calls it.
 *
 * Parity pinning: every function here is checked bit-for-bit against the real
 * reference compiled from its own sources (oracle/_ref/libcoalbench_ref.so, see
 * oracle/Makefile) and against the SPEC.md hand examples (tests/test_oracle.py,
 * tests/golden/).
 */
#ifndef FSBM_COAL_ORACLE_H
#define FSBM_COAL_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_NCAT 6

/* status codes (same numbering as include/fsbm_coal.h) */
enum { ORC_OK = 0, ORC_DOMAIN = 1, ORC_SHAPE = 2, ORC_CONFIG = 3, ORC_STIFF = 4 };

/* proj/src/mass_grid.cpp:10-25 */
int orc_mass_grid(int nkr, double x1, double ratio, double *x);
/* proj/src/mass_grid.cpp:27-48 */
int orc_exponential_init(int nkr, const double *x, double n_total, double xbar, double *out);
/* proj/src/coalescence.cpp:36-67 (GainTable ctor); arrays are [i*nkr+j] */
int orc_gain_table(int nkr, const double *x, double ratio, int32_t *lo, double *w_lo,
                   double *w_hi, double *top);
/* proj/src/kernels.cpp:65-93 -> abd[3*p+{0,1,2}] = {source_a, source_b, dest}; returns 20 */
int orc_default_registry(int *abd);
/* proj/src/kernels.cpp:117-140 (family: 0 constant, 1 golovin, 2 product, 3 hydrodynamic) */
int orc_build_tables(int nkr, const double *x, int npairs, int family, double coeff,
                     double level_scale, double pair_scale_step, double *t750, double *t500);
/* proj/include/coalbench/kernels.hpp:123-135 */
double orc_pressure_weight(double pressure);
double orc_interpolate(double k750, double k500, double w);

/* proj/src/coalescence.cpp:204-339.  bins[c] -> nkr doubles of category c (in place).
 * kernel_strategy: 0 precomputed, 1 on_demand.  counters (may be NULL) get
 * += {triples, points, kernel_evals}.  On stiffness returns ORC_STIFF with
 * err_cat/err_bin set; bins are then partially updated exactly like the reference. */
int orc_coal_step(int nkr, const double *x, int npairs, const int *abd, const double *t750,
                  const double *t500, const int32_t *g_lo, const double *g_wlo,
                  const double *g_whi, const double *g_top, double *const bins[ORC_NCAT],
                  double pressure, double dt, int substeps, int kernel_strategy,
                  uint64_t *counters, int *err_cat, int *err_bin);

/* proj/include/coalbench/rng.hpp:10-32 */
uint64_t orc_splitmix_next(uint64_t *state);
double orc_uniform01(uint64_t *state);
uint64_t orc_bounded(uint64_t *state, uint64_t bound);

/* proj/src/driver.cpp:223-285 (make_synthetic_case). bins: category-major [6][np*nkr]. */
int orc_synthetic_case(int ni, int nk, int nj, double cloud_fraction, uint64_t seed, int nkr,
                       double x1, double ratio, double number_density, double *temperature,
                       double *pressure, double *bins);

/* SURVEY.md 8(d) "thunderstorm" spectra for one mask-true point at linear index p:
 * category c gets exponential_init(grid, 1e6*(0.5+u_c)*s_c, x[min(nkr-1, nkr/3 + c*nkr/16)])
 * with s = {1, 1/4, 1/4, 1/4, 1/4, 1/4} and u_c the c-th uniform01() draw of
 * SplitMix64(seed ^ p).  out: [6][nkr]. */
int orc_thunderstorm_point(int nkr, const double *x, uint64_t seed, uint64_t p, double *out);

/* orc_thunderstorm_point for points p0..p0+n-1 where mask (nullable) is set;
 * others zeroed.  bins category-major [6][n*nkr]. */
int orc_thunderstorm_block(int nkr, const double *x, uint64_t seed, uint64_t p0, uint64_t n,
                           const uint8_t *mask, double *bins);

/* proj/src/driver.cpp:198-211 */
uint64_t orc_fission_predicates(uint64_t npoints, const double *temperature, uint8_t *mask);

/* Phase 2 of fissioned_step (proj/src/driver.cpp:384-430) over a whole (i,k,j)
 * domain, serial (j,k,i) order, one whole-domain tile.  bins category-major
 * [6][np*nkr].  Stops at the first stiffness error (err5 = {cat, bin, i, k, j},
 * 1-based i,k,j) exactly like the serial reference.  nthreads>1 splits the
 * flattened (j,k,i) range into contiguous chunks (run_chunks, driver.cpp:56-84). */
int orc_step_grid(int ni, int nk, int nj, int nkr, const double *x, int npairs, const int *abd,
                  const double *t750, const double *t500, const int32_t *g_lo,
                  const double *g_wlo, const double *g_whi, const double *g_top,
                  const uint8_t *mask, const double *pressure, double *bins, double dt,
                  int substeps, int kernel_strategy, int nthreads, uint64_t *counters,
                  int *err5);

/* ---- Bott (1998) flux method, multi-category FSBM form (oracle/bott_oracle.c) ----
 * No reference implementation exists: pinned by known-answer tests. */
/* Courant numbers [i*nkr+j] of the flux targets g_lo (GainTable lo; 0 for top cells). */
int orc_bott_courant(int nkr, const double *x, const int32_t *g_lo, double *cour);
/* Bott's eq. 13 flux of gsk from bin k (after the gain: gk) into bin k+1 (gkp). */
double orc_bott_flux(double gsk, double gk, double gkp, double c);
/* One coal step with Bott's flux method instead of Kovetz-Olund; same inputs, counters
 * and registry semantics as orc_coal_step.  Never raises stiffness (positive-definite). */
int orc_bott_step(int nkr, const double *x, int npairs, const int *abd, const double *t750,
                  const double *t500, const int32_t *g_lo, const double *cour,
                  double *const bins[ORC_NCAT], double pressure, double dt, int substeps,
                  int kernel_strategy, uint64_t *counters);
/* orc_bott_step at every mask-true point (mask nullable) of np points; bins category-major
 * [6][np*nkr]; nthreads contiguous point ranges. */
int orc_bott_step_grid(size_t np, int nkr, const double *x, int npairs, const int *abd,
                       const double *t750, const double *t500, const int32_t *g_lo,
                       const double *cour, const uint8_t *mask, const double *pressure,
                       double *bins, double dt, int substeps, int kernel_strategy, int nthreads,
                       uint64_t *counters);

#ifdef __cplusplus
}
#endif
#endif
