// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (oracle side).
//
// A thin extern "C" shim over the *unmodified* reference library
// (/root/reference/proj/src/{mass_grid,kernels,coalescence,driver,snapshot,verify}.cpp),
// compiled by oracle/Makefile into oracle/_ref/libcoalbench_ref.so.  It lets
// the parity tests and bench.py's CPU-baseline leg call the real reference
// (`coal_step`, `fissioned_step`, `GainTable`, `build_tables`, ...) on the
// same input bytes as the CUDA path.  Nothing in the product links this.
//
// Status codes mirror include/fsbm_coal.h: 0 ok, 1 domain, 2 shape,
// 3 config, 4 stiffness, 5 allocation, 7 other.

#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "coalbench/coalescence.hpp"
#include "coalbench/driver.hpp"
#include "coalbench/errors.hpp"
#include "coalbench/kernels.hpp"
#include "coalbench/mass_grid.hpp"
#include "coalbench/snapshot.hpp"
#include "coalbench/verify.hpp"

using namespace coalbench;

namespace {

thread_local std::string g_last_error;

int status_of(const std::exception& e) {
    g_last_error = e.what();
    if (dynamic_cast<const StiffnessError*>(&e)) return 4;
    if (dynamic_cast<const AllocationError*>(&e)) return 5;
    if (dynamic_cast<const ShapeError*>(&e)) return 2;
    if (dynamic_cast<const ConfigError*>(&e)) return 3;
    if (dynamic_cast<const DomainError*>(&e)) return 1;
    return 7;
}

PairRegistry registry_from(int npairs, const int* abd) {
    if (abd == nullptr) return default_pair_registry();
    PairRegistry r;
    for (int p = 0; p < npairs; ++p)
        r.push_back({"p" + std::to_string(p), static_cast<Category>(abd[3 * p]),
                     static_cast<Category>(abd[3 * p + 1]), static_cast<Category>(abd[3 * p + 2])});
    return r;
}

KernelTableSet tables_from(int nkr, int npairs, const int* abd, const double* t750,
                           const double* t500) {
    KernelTableSet t(nkr, registry_from(npairs, abd));
    const int np = t.num_pairs();
    for (int p = 0; p < np; ++p)
        for (int i = 0; i < nkr; ++i)
            for (int j = 0; j < nkr; ++j) {
                const std::size_t idx = (static_cast<std::size_t>(p) * nkr + i) * nkr + j;
                t.mutable_750(p, i, j) = t750[idx];
                t.mutable_500(p, i, j) = t500[idx];
            }
    return t;
}

} // namespace

extern "C" {

const char* cbref_last_error(void) { return g_last_error.c_str(); }

int cbref_default_registry(int* abd) {
    PairRegistry r = default_pair_registry();
    for (std::size_t p = 0; p < r.size(); ++p) {
        abd[3 * p] = static_cast<int>(r[p].source_a);
        abd[3 * p + 1] = static_cast<int>(r[p].source_b);
        abd[3 * p + 2] = static_cast<int>(r[p].dest);
    }
    return static_cast<int>(r.size());
}

int cbref_mass_grid(int nkr, double x1, double ratio, double* x_out) {
    try {
        MassGrid g = make_mass_grid(nkr, x1, ratio);
        std::memcpy(x_out, g.x.data(), sizeof(double) * nkr);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int cbref_gain_table(int nkr, double x1, double ratio, int* lo, double* w_lo, double* w_hi,
                     double* top) {
    try {
        MassGrid g = make_mass_grid(nkr, x1, ratio);
        GainTable gt(g);
        for (int i = 0; i < nkr; ++i)
            for (int j = 0; j < nkr; ++j) {
                const auto& e = gt.at(i, j);
                const std::size_t k = static_cast<std::size_t>(i) * nkr + j;
                lo[k] = e.lo;
                w_lo[k] = e.w_lo;
                w_hi[k] = e.w_hi;
                top[k] = e.top_factor;
            }
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int cbref_build_tables(int nkr, double x1, double ratio, int npairs, const int* abd, int family,
                       double coeff, double level_scale, double pair_scale_step, double* t750,
                       double* t500) {
    try {
        MassGrid g = make_mass_grid(nkr, x1, ratio);
        KernelParams kp;
        kp.family = static_cast<KernelFamily>(family);
        kp.coeff = coeff;
        kp.level_scale = level_scale;
        kp.pair_scale_step = pair_scale_step;
        KernelTableSet t = build_tables(g, registry_from(npairs, abd), kp);
        for (int p = 0; p < t.num_pairs(); ++p)
            for (int i = 0; i < nkr; ++i)
                for (int j = 0; j < nkr; ++j) {
                    const std::size_t idx = (static_cast<std::size_t>(p) * nkr + i) * nkr + j;
                    t750[idx] = t.value_750(p, i, j);
                    t500[idx] = t.value_500(p, i, j);
                }
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int cbref_exponential_init(int nkr, double x1, double ratio, double n_total, double xbar,
                           double* out) {
    try {
        MassGrid g = make_mass_grid(nkr, x1, ratio);
        BinDistribution d = exponential_init(g, n_total, xbar);
        std::memcpy(out, d.n.data(), sizeof(double) * nkr);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

double cbref_pressure_weight(double p) { return pressure_weight(p); }

/// kernel_at for one entry (adds 1 to the table's counter, which is discarded).
int cbref_kernel_at(int nkr, int npairs, const int* abd, const double* t750, const double* t500,
                    int pair, int i, int j, double pressure, double* out) {
    try {
        KernelTableSet t = tables_from(nkr, npairs, abd, t750, t500);
        *out = kernel_at(t, pair, i, j, pressure);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

/// coal_step on one point. bins6 is category-major: bins6[c*nkr + k].
/// counters_out = {triples, points, kernel_evals}; err_out = {category, bin}.
int cbref_coal_step(int nkr, double x1, double ratio, int npairs, const int* abd,
                    const double* t750, const double* t500, double* bins6, double pressure,
                    double dt, int substeps, int kernel_strategy, int scratch_strategy,
                    uint64_t* counters_out, int* err_out) {
    try {
        MassGrid g = make_mass_grid(nkr, x1, ratio);
        KernelTableSet t = tables_from(nkr, npairs, abd, t750, t500);
        GainTable gt(g);
        CoalCounters cc;
        CoalContext ctx{&g, &t, &gt, &cc};
        CoalConfig cfg;
        cfg.dt = dt;
        cfg.substeps = substeps;
        cfg.kernel_strategy =
            kernel_strategy == 0 ? KernelStrategy::precomputed : KernelStrategy::on_demand;
        cfg.scratch_strategy =
            scratch_strategy == 0 ? ScratchStrategy::automatic : ScratchStrategy::arena;
        PointState ps;
        for (int c = 0; c < kNumCategories; ++c)
            ps.n[c] = std::span<double>(bins6 + static_cast<std::size_t>(c) * nkr, nkr);
        std::vector<double> sbuf(static_cast<std::size_t>(2 * kNumCategories) * nkr);
        ScratchSlice slice;
        for (int c = 0; c < kNumCategories; ++c) {
            slice.work[c] = std::span<double>(sbuf.data() + c * nkr, nkr);
            slice.delta[c] = std::span<double>(sbuf.data() + (kNumCategories + c) * nkr, nkr);
        }
        int st = 0;
        try {
            coal_step(ps, pressure, cfg, ctx, scratch_strategy == 0 ? nullptr : &slice, nullptr);
        } catch (const StiffnessError& e) {
            if (err_out) {
                err_out[0] = e.category();
                err_out[1] = e.bin();
            }
            g_last_error = e.what();
            st = 4;
        }
        if (counters_out) {
            counters_out[0] = cc.triples.load();
            counters_out[1] = cc.points.load();
            counters_out[2] = t.eval_count();
        }
        return st;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

/// make_synthetic_case; bins is category-major [6][npoints*nkr].
int cbref_synthetic_case(int ni, int nk, int nj, double cloud_fraction, uint64_t seed, int nkr,
                         double x1, double ratio, double number_density, double* temperature,
                         double* pressure, double* bins) {
    try {
        SyntheticCaseParams sp;
        sp.ni = ni;
        sp.nk = nk;
        sp.nj = nj;
        sp.cloud_fraction = cloud_fraction;
        sp.seed = seed;
        sp.nkr = nkr;
        sp.x1 = x1;
        sp.ratio = ratio;
        sp.number_density = number_density;
        GridState s = make_synthetic_case(sp);
        const std::size_t np = s.ranges.npoints();
        std::memcpy(temperature, s.temperature.data(), sizeof(double) * np);
        std::memcpy(pressure, s.pressure.data(), sizeof(double) * np);
        for (int c = 0; c < kNumCategories; ++c)
            std::memcpy(bins + static_cast<std::size_t>(c) * np * nkr, s.bins[c].data(),
                        sizeof(double) * np * nkr);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

/// fission_predicates; returns true_count via *count.
int cbref_fission_predicates(int ni, int nk, int nj, const double* temperature, uint8_t* mask,
                             uint64_t* count) {
    try {
        GridState s;
        s.ranges = Ranges{1, ni, 1, nk, 1, nj};
        s.grid = make_mass_grid(2, 1.0, 2.0);
        s.temperature.assign(temperature, temperature + s.ranges.npoints());
        PredicateMask m = fission_predicates(s);
        std::memcpy(mask, m.call_coal.data(), m.call_coal.size());
        *count = m.true_count;
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

/// One fissioned_step (stubs disabled) over host arrays, in place.
/// plan: mode 0 serial / 1 parallel; collapse 2|3; kernel 0 precomputed / 1 on_demand;
/// scratch 0 automatic / 1 arena.  counters_out = {triples, points, kernel_evals};
/// timings_out = {coal_s, step_s}; err_out = {category, bin, i, k, j}.
int cbref_fissioned_step(int ni, int nk, int nj, int nkr, double x1, double ratio, int npairs,
                         const int* abd, const double* t750, const double* t500,
                         const double* temperature, const double* pressure, double* bins,
                         double dt, int substeps, int mode, int collapse, int threads,
                         int kernel_strategy, int scratch_strategy, int n_patches, int n_tiles,
                         uint64_t* counters_out, double* timings_out, int* err_out) {
    try {
        GridState s;
        s.ranges = Ranges{1, ni, 1, nk, 1, nj};
        s.grid = make_mass_grid(nkr, x1, ratio);
        const std::size_t np = s.ranges.npoints();
        s.temperature.assign(temperature, temperature + np);
        s.pressure.assign(pressure, pressure + np);
        for (int c = 0; c < kNumCategories; ++c)
            s.bins[c].assign(bins + static_cast<std::size_t>(c) * np * nkr,
                             bins + static_cast<std::size_t>(c + 1) * np * nkr);
        KernelTableSet t = tables_from(nkr, npairs, abd, t750, t500);
        GainTable gt(s.grid);
        PredicateMask mask = fission_predicates(s);
        ExecPlan plan;
        plan.mode = mode == 0 ? StepMode::serial : StepMode::parallel;
        plan.collapse = collapse;
        plan.threads = threads;
        plan.kernel_strategy =
            kernel_strategy == 0 ? KernelStrategy::precomputed : KernelStrategy::on_demand;
        plan.scratch_strategy =
            scratch_strategy == 0 ? ScratchStrategy::automatic : ScratchStrategy::arena;
        std::vector<ScratchArena> arena;
        if (plan.scratch_strategy == ScratchStrategy::arena)
            arena.push_back(allocate_arena(ni, nk, nj, nkr, ScratchArena::kIceMax));
        WorkCounters wc;
        PhaseTimings pt;
        PatchTilePlan tiles;
        const bool use_tiles = n_patches > 1 || n_tiles > 1;
        if (use_tiles) tiles = decompose(s.ranges, n_patches, n_tiles);
        StepContext ctx;
        ctx.tables = &t;
        ctx.gains = &gt;
        ctx.coal.dt = dt;
        ctx.coal.substeps = substeps;
        ctx.stubs.nucleation_iters = 0;
        ctx.stubs.condensation_iters = 0;
        ctx.arena = arena.empty() ? nullptr : &arena[0];
        ctx.counters = &wc;
        ctx.timings = &pt;
        ctx.tiles = use_tiles ? &tiles : nullptr;
        int st = 0;
        try {
            fissioned_step(s, mask, ctx, plan);
        } catch (const StiffnessError& e) {
            if (err_out) {
                err_out[0] = e.category();
                err_out[1] = e.bin();
                err_out[2] = e.i();
                err_out[3] = e.k();
                err_out[4] = e.j();
            }
            g_last_error = e.what();
            st = 4;
        }
        for (int c = 0; c < kNumCategories; ++c)
            std::memcpy(bins + static_cast<std::size_t>(c) * np * nkr, s.bins[c].data(),
                        sizeof(double) * np * nkr);
        if (counters_out) {
            counters_out[0] = wc.coal.triples.load();
            counters_out[1] = wc.coal.points.load();
            counters_out[2] = t.eval_count();
        }
        if (timings_out) {
            timings_out[0] = pt.coal_s;
            timings_out[1] = pt.step_s;
        }
        return st;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

namespace {
GridState state_from(const int* rg, int nkr, double ratio, const double* x, const double* T,
                     const double* P, const double* bins) {
    GridState s;
    s.ranges = Ranges{rg[0], rg[1], rg[2], rg[3], rg[4], rg[5]};
    s.grid.x.assign(x, x + nkr);
    s.grid.ratio = ratio;
    const std::size_t np = s.ranges.npoints();
    s.temperature.assign(T, T + np);
    s.pressure.assign(P, P + np);
    for (int c = 0; c < kNumCategories; ++c)
        s.bins[c].assign(bins + static_cast<std::size_t>(c) * np * nkr,
                         bins + static_cast<std::size_t>(c + 1) * np * nkr);
    return s;
}
} // namespace

/// write_snapshot of a state given as ranges[6], x[nkr], T/P[np], bins[6*np*nkr].
int cbref_write_snapshot(const char* path, const int* ranges, int nkr, double ratio,
                         const double* x, const double* T, const double* P, const double* bins) {
    try {
        write_snapshot(state_from(ranges, nkr, ratio, x, T, P, bins), path);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

/// read_snapshot: call with bins == nullptr to get ranges[6]/nkr/ratio only.
int cbref_read_snapshot(const char* path, int* ranges, int* nkr, double* ratio, double* x,
                        double* T, double* P, double* bins) {
    try {
        GridState s = read_snapshot(path);
        const Ranges& r = s.ranges;
        const int rv[6] = {r.ids, r.ide, r.kds, r.kde, r.jds, r.jde};
        std::memcpy(ranges, rv, sizeof(rv));
        *nkr = s.nkr();
        *ratio = s.grid.ratio;
        if (bins) {
            const std::size_t np = r.npoints();
            std::memcpy(x, s.grid.x.data(), sizeof(double) * s.nkr());
            std::memcpy(T, s.temperature.data(), sizeof(double) * np);
            std::memcpy(P, s.pressure.data(), sizeof(double) * np);
            for (int c = 0; c < kNumCategories; ++c)
                std::memcpy(bins + static_cast<std::size_t>(c) * np * s.nkr(), s.bins[c].data(),
                            sizeof(double) * np * s.nkr());
        }
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int cbref_digit_agreement(double a, double b, int* digits) {
    try {
        *digits = digit_agreement(a, b);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

/// compare_states over two states of the same ranges/nkr; per field (9, the
/// reference's order): min_digits, mean_digits, count_compared, count_exact.
int cbref_compare_states(const int* ranges, int nkr, const double* xa, const double* Ta,
                         const double* Pa, const double* binsa, const double* xb,
                         const double* Tb, const double* Pb, const double* binsb, int* min_d,
                         double* mean_d, uint64_t* compared, uint64_t* exact) {
    try {
        DiffReport r = compare_states(state_from(ranges, nkr, 2.0, xa, Ta, Pa, binsa),
                                      state_from(ranges, nkr, 2.0, xb, Tb, Pb, binsb));
        for (std::size_t f = 0; f < r.fields.size(); ++f) {
            min_d[f] = r.fields[f].min_digits;
            mean_d[f] = r.fields[f].mean_digits;
            compared[f] = r.fields[f].count_compared;
            exact[f] = r.fields[f].count_exact;
        }
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

} // extern "C"
