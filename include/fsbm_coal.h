/* fsbm_coal.h -- C ABI of the B200-native FSBM collision-coalescence hot path.
 *
 * Drop-in boundary for the reference mini-app `coalbench`
 * (/root/reference/proj).  Every entry point names the reference interface it
 * replaces.  Plain pointers and sizes only; no exceptions cross the ABI: every
 * function returns an fsbm_status and fsbm_last_error() holds the message.
 *
 * Data layout is the reference's GridState (driver.hpp:40-61): six separate
 * category arrays bins[c][point*nkr + bin] with point = ((i-ids)*nk + (k-kds))*nj
 * + (j-jds) (i slowest, j fastest, bin innermost); temperature/pressure are
 * [npoints].  Category order liquid, ice1, ice2, ice3, snow, graupel
 * (kernels.hpp:17-26).
 */
#ifndef FSBM_COAL_H
#define FSBM_COAL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSBM_NCAT 6
#define FSBM_ABI_VERSION 2

/* Error taxonomy of errors.hpp:10-74 as status codes. */
typedef enum {
    FSBM_OK = 0,
    FSBM_DOMAIN = 1,    /* DomainError    (errors.hpp:17-20) */
    FSBM_SHAPE = 2,     /* ShapeError     (errors.hpp:23-26) */
    FSBM_CONFIG = 3,    /* ConfigError    (errors.hpp:29-32) */
    FSBM_STIFFNESS = 4, /* StiffnessError (errors.hpp:35-62) */
    FSBM_ALLOC = 5,     /* AllocationError(errors.hpp:65-74) */
    FSBM_CUDA = 6,      /* device/runtime failure (no reference analogue) */
    FSBM_INTERNAL = 7
} fsbm_status;

/* coalbench::Ranges (driver.hpp:23-35): inclusive, 1-based as in WRF. */
typedef struct {
    int ids, ide, kds, kde, jds, jde;
} fsbm_ranges;

/* coalbench::ExecPlan (driver.hpp:103-109) + the numerics mode.
 * mode: 0 serial, 1 parallel; collapse: 2 or 3; threads >= 1 (validated exactly
 * as validate_plan, driver.cpp:213-221; the device ignores them -- scheduling
 * never changes results); kernel_strategy: 0 precomputed, 1 on_demand (changes
 * only the kernel_evals counter, kernels.cpp:154-172); scratch_strategy:
 * 0 automatic, 1 arena.  numerics: FSBM_NUMERICS_FAST (FP64, reassociated
 * sums; <=1e-12 relative per bin vs the reference) or FSBM_NUMERICS_EXACT
 * (bitwise identical to coal_step: same operation order, no FMA).
 * FSBM_NUMERICS_BOTT replaces the Kovetz-Olund split by Bott's (1998) flux method (the
 * WRF coal_bott_new scheme the reference declares out of scope): same
 * inputs, registry order and counters; positive-definite (never FSBM_STIFFNESS);
 * checked against oracle/bott_oracle.c. */
enum { FSBM_PRECOMPUTED = 0, FSBM_ON_DEMAND = 1 };
enum { FSBM_AUTOMATIC = 0, FSBM_ARENA = 1 };
enum { FSBM_NUMERICS_FAST = 0, FSBM_NUMERICS_EXACT = 1, FSBM_NUMERICS_BOTT = 2 };
typedef struct {
    int mode;
    int collapse;
    int threads;
    int kernel_strategy;
    int scratch_strategy;
    int numerics;
} fsbm_plan;

/* PatchTilePlan::Tile (driver.hpp:69-80), listed in patch-major, tile-minor
 * order.  Only affects which point a StiffnessError reports (the first failing
 * point in (tile, j, k, i) order, as run_chunks/fissioned_step would). */
typedef struct {
    int its, ite, jts, jte;
} fsbm_tile;

/* CoalCounters (coalescence.hpp:68-71) + KernelTableSet::eval_count
 * (kernels.hpp:101-102): triples = (pair,i,j) visits, points = coal_step calls. */
typedef struct {
    uint64_t triples;
    uint64_t points;
    uint64_t kernel_evals;
} fsbm_counters;

/* StiffnessError (errors.hpp:35-62) incl. at_point (1-based i,k,j) and the negative
 * value the reference prints in its message (coalescence.cpp:319-325). */
typedef struct {
    int category, bin;
    int has_point;
    int i, k, j;
    double value;
} fsbm_error;

typedef struct fsbm_ctx fsbm_ctx; /* opaque: device tables, gain table, registry */

const char *fsbm_last_error(void);
int fsbm_abi_version(void);

/* Replaces the setup of StepContext{tables, gains} (driver.hpp:141-150):
 * KernelTableSet (kernels.hpp:81-114, t750/t500 laid out [pair][i][j] as
 * kernels.hpp:105-107), the registry (kernels.hpp:33-50; abd[3p..3p+2] =
 * source_a, source_b, dest) and GainTable(grid) (coalescence.cpp:36-67, built
 * here bit-identically from x[] and ratio, MassGrid mass_grid.hpp:9-14).
 * Uploads everything to `device` once; no allocation happens per step. */
int fsbm_ctx_create(int device, int nkr, const double *x, double ratio, int npairs,
                    const int *pair_abd, const double *t750, const double *t500,
                    fsbm_ctx **out);
int fsbm_ctx_destroy(fsbm_ctx *ctx);

/* GainTable::at(i,j) (coalescence.hpp:58) for the whole nkr x nkr table, as
 * built by fsbm_ctx_create (flux-target selection; bit-exact contract). */
int fsbm_ctx_gain_table(const fsbm_ctx *ctx, int32_t *lo, double *w_lo, double *w_hi,
                        double *top);

/* fission_predicates (driver.cpp:198-211) on device: mask[p] = T>193.15 &&
 * T>223.15; *count = true_count.  stream may be NULL (legacy default stream). */
int fsbm_fission_predicates_device(fsbm_ctx *ctx, size_t npoints, const double *temperature_d,
                                   uint8_t *mask_d, uint64_t *count, void *stream);

/* Phase 2 of fissioned_step (driver.cpp:353-434, driver.hpp:179-180) on
 * DEVICE buffers: coal_step (coalescence.cpp:204-339) at exactly the mask-true
 * points, in place.  temperature_d is used for the stale-mask check
 * (driver.cpp:361-367) and may be NULL to skip it; mask_d may be NULL to derive
 * it from temperature_d.  tiles may be NULL (whole domain).  counters_out (may
 * be NULL) receives this call's counts; err_out (may be NULL) is filled on
 * FSBM_STIFFNESS with the first failing point in (tile, j, k, i) order.  The
 * call is stream-ordered but synchronises once at the end to report status.
 * After FSBM_STIFFNESS the state is unspecified (the reference leaves it
 * partially mutated too). */
int fsbm_step_grid_device(fsbm_ctx *ctx, fsbm_ranges ranges, double *const bins_d[FSBM_NCAT],
                          const double *pressure_d, const double *temperature_d,
                          const uint8_t *mask_d, double dt, int substeps, const fsbm_plan *plan,
                          const fsbm_tile *tiles, int ntiles, void *stream,
                          fsbm_counters *counters_out, fsbm_error *err_out);

/* Same on HOST buffers (the reference's GridState vectors): H2D of the state,
 * the step, D2H of the bins -- pipelined in chunks over i-slabs so copies
 * overlap compute.  Pinned host memory is fastest but not required. */
int fsbm_step_grid_host(fsbm_ctx *ctx, fsbm_ranges ranges, double *const bins_h[FSBM_NCAT],
                        const double *pressure_h, const double *temperature_h,
                        const uint8_t *mask_h, double dt, int substeps, const fsbm_plan *plan,
                        const fsbm_tile *tiles, int ntiles, fsbm_counters *counters_out,
                        fsbm_error *err_out);

/* fsbm_step_grid_host on the patch `patch` (global 1-based extents, an i/j sub-range with
 * all of k) of a host GridState whose arrays span `global`: the caller passes the GLOBAL
 * arrays, the H2D/D2H copies are pitched (one (i,k) line of the patch per row), so a
 * WRF-style j-patch (decompose, driver.cpp:187-196) is stepped in place without a
 * host-side gather.  fsbm_step_grid_host(r) == fsbm_step_patch_host(r, r). */
int fsbm_step_patch_host(fsbm_ctx *ctx, fsbm_ranges global, fsbm_ranges patch,
                         double *const bins_h[FSBM_NCAT], const double *pressure_h,
                         const double *temperature_h, const uint8_t *mask_h, double dt,
                         int substeps, const fsbm_plan *plan, const fsbm_tile *tiles, int ntiles,
                         fsbm_counters *counters_out, fsbm_error *err_out);

/* Diagnostics of a device state: out[c] = sum of n over all points and bins of category c,
 * out[6 + c] = sum of n*x[bin] (total_number / total_mass, mass_grid.hpp, summed over the
 * grid; deterministic order for a given npoints).  Synchronises `stream`. */
int fsbm_state_moments_device(fsbm_ctx *ctx, size_t npoints, const double *const bins_d[FSBM_NCAT],
                              double out[2 * FSBM_NCAT], void *stream);

/* coal_step (coalescence.hpp:148-150) for ONE point on host spans (bins6 is
 * category-major [6][nkr]); a one-point launch.  Error semantics as coal_step
 * (DomainError on dt<=0 / substeps<1). */
int fsbm_coal_step(fsbm_ctx *ctx, double *bins6, double pressure, double dt, int substeps,
                   int kernel_strategy, int numerics, fsbm_counters *counters_out,
                   fsbm_error *err_out);

/* ---- synthetic inputs (bench / parity fixtures; not part of the step) ---- */

/* make_synthetic_case's temperature/pressure recipe (driver.cpp:223-272) on the
 * host: exactly round(cf*N) cloudy points chosen by a SplitMix64 Fisher-Yates
 * shuffle, cloudy T = 240+60u, others 210/180 K, pressure 900->400 hPa in k.
 * liquid_init (nullable, [npoints*nkr]) receives the reference's liquid-only
 * spectra (driver.cpp:274-283) for cloudy points. */
int fsbm_synth_thermo_host(int ni, int nk, int nj, double cloud_fraction, uint64_t seed,
                           int nkr, const double *x, double number_density,
                           double *temperature, double *pressure, double *liquid_init);

/* SURVEY 8(d) "thunderstorm" spectra for every mask-true point, generated on
 * device (counter-based: SplitMix64(seed ^ (point_offset + p))); all six
 * categories; mask-false points are zeroed.  point_offset is the global linear
 * index of local point 0, so a shard reproduces its slice of the full domain. */
int fsbm_synth_thunderstorm_device(fsbm_ctx *ctx, size_t npoints, uint64_t point_offset,
                                   const uint8_t *mask_d, uint64_t seed,
                                   double *const bins_d[FSBM_NCAT], void *stream);

/* Device time (CUDA events on the launching stream) of the coalescence kernel in
 * the most recent fsbm_step_grid_* call on this context, in milliseconds, and
 * the number of this library's kernels that call launched. */
int fsbm_ctx_last_timing(const fsbm_ctx *ctx, float *coal_kernel_ms, int *launches);

/* Which FSBM_NUMERICS_FAST kernel this context dispatches to: 1 coal_fast (direct
 * FP64, any nkr), 2 coal_dmma (FP64 tensor cores, nkr 32/33), 3 coal_dmmag (FP64
 * tensor cores, general band grids up to ~190 bins).  FSBM_FAST_KERNEL=direct|dmma|dmmag
 * in the environment at fsbm_ctx_create forces one (A/B and parity testing). */
int fsbm_ctx_fast_kernel(const fsbm_ctx *ctx, int *kernel);

/* Measured FP64 roof of `device`: a DFMA-chain microbenchmark (8 independent
 * chains per thread, full occupancy) timed with CUDA events; FLOP/s counts 2 per
 * DFMA.  MEASURED_PEAKS.json carries HBM and bf16 only, so the bench measures
 * the denominator of its FP64 roofline live with this. */
int fsbm_probe_fp64_peak(int device, double *tflops);

/* ---- state snapshots and the digit-agreement comparator ---- */

/* write_snapshot (snapshot.hpp:8-17, snapshot.cpp:46-73): the CBSNAP01 layout
 * (magic, u32 version 1, u32 nkr, i32 ids..jde, f64 ratio, u32 ncat + names,
 * f64 x[nkr], temperature[np], pressure[np], 6 x bins[np*nkr]), little-endian,
 * bit-exact on round trip.  Host arrays in GridState layout. */
int fsbm_snapshot_write(const char *path, fsbm_ranges ranges, int nkr, double ratio,
                        const double *x, const double *temperature, const double *pressure,
                        const double *const bins[FSBM_NCAT]);

/* read_snapshot (snapshot.cpp:75-135) in two calls: the header, then the arrays into
 * caller buffers sized from it.  FSBM_CONFIG (ConfigError) on a malformed, truncated or
 * over-long file, with the reference's messages and check order. */
int fsbm_snapshot_read_header(const char *path, fsbm_ranges *ranges, int *nkr, double *ratio);
int fsbm_snapshot_read(const char *path, double *x, double *temperature, double *pressure,
                       double *const bins[FSBM_NCAT]);

/* FieldDiff (verify.hpp:20-26). */
typedef struct {
    int min_digits;
    double mean_digits;
    uint64_t count_compared;
    uint64_t count_exact;
} fsbm_field_diff;

/* compare_states (verify.cpp:65-80) on DEVICE arrays of two states of the same shape
 * (the caller checks ranges/nkr -> ShapeError): out[9] = mass_grid, temperature,
 * pressure, liquid..graupel, each the digit_agreement (verify.cpp:12-26) min / mean /
 * exact count over its values, one reduction launch.  FSBM_DOMAIN on a non-finite
 * value (digit_agreement throws DomainError). */
int fsbm_compare_states_device(int device, size_t npoints, int nkr, const double *x_a,
                               const double *temperature_a, const double *pressure_a,
                               const double *const bins_a[FSBM_NCAT], const double *x_b,
                               const double *temperature_b, const double *pressure_b,
                               const double *const bins_b[FSBM_NCAT], fsbm_field_diff *out,
                               void *stream);

/* ---- multi-GPU: shards, device groups, NCCL diagnostics ----
 *
 * Microphysics is column-local: shards are independent, there is no halo and no
 * data-path collective.  A group owns one context per local device and steps each local
 * shard from its own host thread; counters, status, the first failing point (serial
 * (tile, j, k, i) order over the whole domain) and diagnostics are combined on the host
 * and, across processes, by one NCCL all-reduce group issued by the library (NCCL is
 * dlopen'ed; single-process groups never load it).  Results per point do not depend on
 * the decomposition in EXACT numerics (bitwise); in FAST numerics a point's rounding can
 * depend on which points share its 16-point group, within the same 1e-12 bar. */
enum { FSBM_SPLIT_I = 0, FSBM_SPLIT_J = 1 };

/* split_range (driver.cpp:35-51) over i (i-slabs) or j (the WRF patches of decompose,
 * driver.cpp:187-196): nshards near-equal ranges, remainder to the first, all k.
 * FSBM_DOMAIN when nshards does not fit the extent (the reference's DomainError). */
int fsbm_decompose(fsbm_ranges global, int nshards, int split, fsbm_ranges *shards_out);

/* 128-byte ncclUniqueId for a multi-process group (rank 0 creates it, the caller
 * broadcasts it, e.g. over torch.distributed or MPI). */
int fsbm_nccl_unique_id(uint8_t id[128]);

typedef struct fsbm_group fsbm_group;

/* ndev local devices (repeats allowed: several shards on one GPU); this process is
 * `rank` of `nranks` processes (1 for a single-process group; nccl_id may then be NULL).
 * Table arguments as fsbm_ctx_create. */
int fsbm_group_create(int ndev, const int *devices, int rank, int nranks, const uint8_t *nccl_id,
                      int nkr, const double *x, double ratio, int npairs, const int *pair_abd,
                      const double *t750, const double *t500, fsbm_group **out);
int fsbm_group_destroy(fsbm_group *group);
/* The context of local device `local` (device allocation, synthetic inputs, timing). */
int fsbm_group_ctx(fsbm_group *group, int local, fsbm_ctx **ctx);

/* One local shard of a device-resident domain: its global extents and its own arrays
 * in GridState layout over those extents. */
typedef struct {
    fsbm_ranges ranges;
    double *bins[FSBM_NCAT];
    const double *pressure, *temperature;
    const uint8_t *mask;
    void *stream;
} fsbm_shard;

/* Reduced over every shard of every rank. */
typedef struct {
    double number_before[FSBM_NCAT], number_after[FSBM_NCAT];
    double mass_before[FSBM_NCAT], mass_after[FSBM_NCAT];
    float coal_kernel_ms_max;
} fsbm_diag;

/* fissioned_step over the group's shards (shards[ndev], device arrays): every output is
 * the whole domain's, identical on every rank -- counters summed, the error that the
 * serial reference would raise (earliest phase first, then the first failing point in
 * (tile, j, k, i) order; tiles in global coordinates).  diag_out (nullable) adds two
 * moment passes per shard. */
int fsbm_group_step_device(fsbm_group *group, const fsbm_shard *shards, double dt, int substeps,
                           const fsbm_plan *plan, const fsbm_tile *tiles, int ntiles,
                           fsbm_counters *counters_out, fsbm_error *err_out, fsbm_diag *diag_out);

/* fissioned_step on a host GridState spanning `global`: split into ndev*nranks i-slabs
 * or j-patches; this process steps shards rank*ndev .. rank*ndev+ndev-1 in place
 * (fsbm_step_patch_host, one host thread per device). */
int fsbm_group_step_host(fsbm_group *group, fsbm_ranges global, int split,
                         double *const bins_h[FSBM_NCAT], const double *pressure_h,
                         const double *temperature_h, const uint8_t *mask_h, double dt,
                         int substeps, const fsbm_plan *plan, const fsbm_tile *tiles, int ntiles,
                         fsbm_counters *counters_out, fsbm_error *err_out);

/* Max over all devices of all ranks of the coalescence kernel time of the last step. */
int fsbm_group_last_timing(const fsbm_group *group, float *coal_kernel_ms_max);

#ifdef __cplusplus
}
#endif
#endif /* FSBM_COAL_H */
