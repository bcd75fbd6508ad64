// test_dropin.cpp -- the C++ drop-in against the unmodified reference, in one binary.
//
// Links the reference's own translation units (mass_grid, kernels, coalescence, driver;
// compiled from /root/reference by integration/Makefile) and gpu_fissioned_step.cpp over
// libfsbm_coal.so.  For each case both coalbench::fissioned_step and
// coalbench::gpu::fissioned_step run on copies of the same GridState:
//   * EXACT numerics: bitwise_equal states (driver.hpp:66), equal counters / kernel evals;
//   * FAST numerics: per bin |gpu - ref| <= 1e-12|ref| + 1e-15 sum_k ref_c[k], equal counters;
//   * the same exception type, coordinates and (EXACT) message for stiffness, stale masks,
//     bad plans and extent mismatches.
// Exit status 0 and "dropin ok" on success.  Needs a CUDA device.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

#include "coalbench/coalescence.hpp"
#include "coalbench/driver.hpp"
#include "coalbench/errors.hpp"
#include "coalbench/kernels.hpp"
#include "coalbench/mass_grid.hpp"
#include "gpu_fissioned_step.hpp"

using namespace coalbench;

namespace {

int g_fail = 0;
#define CHECK(cond, ...)                                                         \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::fprintf(stderr, "FAIL %s:%d: %s -- ", __FILE__, __LINE__, #cond); \
            std::fprintf(stderr, __VA_ARGS__);                                   \
            std::fprintf(stderr, "\n");                                          \
            ++g_fail;                                                            \
        }                                                                        \
    } while (0)

/// All six categories populated at warm points (the SURVEY 8(d) headline input shape),
/// from the reference's own exponential_init.
void fill_all_categories(GridState& s, std::uint64_t seed) {
    const int nkr = s.nkr();
    for (std::size_t p = 0; p < s.ranges.npoints(); ++p) {
        const double t = s.temperature[p];
        if (!(t > kOuterGateK && t > kCoalGateK)) continue;
        for (int c = 0; c < kNumCategories; ++c) {
            const double u = static_cast<double>(((p + 1) * 2654435761ull ^ seed ^ (c * 97)) % 1000) / 1000.0;
            const int kb = std::min(nkr - 1, nkr / 3 + c * nkr / 16);
            const auto d = exponential_init(s.grid, 1e6 * (0.5 + u) * (c == 0 ? 1.0 : 0.25), s.grid.x[kb]);
            for (int k = 0; k < nkr; ++k) s.bins[c][p * nkr + k] = d.n[k];
        }
    }
}

struct Outcome {
    std::string type, what;
    int cat = -1, bin = -1, i = 0, k = 0, j = 0;
};

Outcome run(const std::function<void()>& f) {
    Outcome o;
    try {
        f();
        o.type = "ok";
    } catch (const StiffnessError& e) {
        o.type = "stiffness";
        o.what = e.what();
        o.cat = e.category();
        o.bin = e.bin();
        if (e.has_point()) {
            o.i = e.i();
            o.k = e.k();
            o.j = e.j();
        }
    } catch (const ConfigError& e) {
        o.type = "config";
        o.what = e.what();
    } catch (const ShapeError& e) {
        o.type = "shape";
        o.what = e.what();
    } catch (const DomainError& e) {
        o.type = "domain";
        o.what = e.what();
    } catch (const Error& e) {
        o.type = "error";
        o.what = e.what();
    }
    return o;
}

bool within_bar(const GridState& got, const GridState& ref, double* worst) {
    const int nkr = ref.nkr();
    bool ok = true;
    *worst = 0.0;
    for (int c = 0; c < kNumCategories; ++c)
        for (std::size_t p = 0; p < ref.ranges.npoints(); ++p) {
            double sum = 0.0;
            for (int k = 0; k < nkr; ++k) sum += std::fabs(ref.bins[c][p * nkr + k]);
            for (int k = 0; k < nkr; ++k) {
                const double r = ref.bins[c][p * nkr + k], g = got.bins[c][p * nkr + k];
                const double tol = 1e-12 * std::fabs(r) + 1e-15 * sum;
                const double e = std::fabs(g - r);
                if (e > tol) ok = false;
                if (tol > 0) *worst = std::max(*worst, e / tol);
            }
        }
    return ok;
}

void compare_case(const char* name, const GridState& s0, const KernelTableSet& tables,
                  const ExecPlan& plan, double dt, int substeps, const PatchTilePlan* tiles,
                  gpu::Numerics numerics) {
    GainTable gains(s0.grid);
    GridState a = s0, b = s0;
    const PredicateMask mask = fission_predicates(s0);
    ScratchArena arena = allocate_arena(s0.ranges.ni(), s0.ranges.nk(), s0.ranges.nj(), s0.nkr(),
                                        ScratchArena::kIceMax);
    WorkCounters ca, cb;
    StepContext ctxa{&tables, &gains, CoalConfig{dt, substeps}, StubParams{0, 0}, &arena, &ca,
                     nullptr, tiles};
    StepContext ctxb = ctxa;
    ctxb.counters = &cb;
    const std::uint64_t e0 = tables.eval_count();
    const Outcome oa = run([&] { fissioned_step(a, mask, ctxa, plan); });
    const std::uint64_t ea = tables.eval_count() - e0;
    gpu::set_options({0, numerics});
    const Outcome ob = run([&] { gpu::fissioned_step(b, mask, ctxb, plan); });
    const std::uint64_t eb = tables.eval_count() - e0 - ea;
    const bool exact = numerics == gpu::Numerics::exact;
    CHECK(oa.type == ob.type, "%s: reference %s (%s) vs gpu %s (%s)", name, oa.type.c_str(),
          oa.what.c_str(), ob.type.c_str(), ob.what.c_str());
    if (oa.type == "ok") {
        if (exact) {
            CHECK(bitwise_equal(a, b), "%s: states differ (exact)", name);
        } else {
            double worst = 0.0;
            CHECK(within_bar(b, a, &worst), "%s: fast numerics out of the bar (%.3g x tol)", name, worst);
        }
        CHECK(ca.coal.triples.load() == cb.coal.triples.load() &&
                  ca.coal.points.load() == cb.coal.points.load() && ea == eb,
              "%s: counters differ (%llu/%llu/%llu vs %llu/%llu/%llu)", name,
              (unsigned long long)ca.coal.triples.load(), (unsigned long long)ca.coal.points.load(),
              (unsigned long long)ea, (unsigned long long)cb.coal.triples.load(),
              (unsigned long long)cb.coal.points.load(), (unsigned long long)eb);
    } else if (oa.type == "stiffness") {
        CHECK(oa.cat == ob.cat && oa.bin == ob.bin && oa.i == ob.i && oa.k == ob.k && oa.j == ob.j,
              "%s: stiffness point differs: ref (%d,%d @ %d,%d,%d) gpu (%d,%d @ %d,%d,%d)", name,
              oa.cat, oa.bin, oa.i, oa.k, oa.j, ob.cat, ob.bin, ob.i, ob.k, ob.j);
        if (exact) CHECK(oa.what == ob.what, "%s: message '%s' vs '%s'", name, oa.what.c_str(), ob.what.c_str());
    }
    std::printf("  %-44s %-5s %-9s %s\n", name, exact ? "exact" : "fast", oa.type.c_str(),
                g_fail ? "(failures so far)" : "ok");
}

} // namespace

int main() {
    const ExecPlan par3{StepMode::parallel, 3, 4, KernelStrategy::on_demand, ScratchStrategy::arena};
    const ExecPlan ser2{StepMode::serial, 2, 1, KernelStrategy::precomputed, ScratchStrategy::automatic};
    for (auto numerics : {gpu::Numerics::exact, gpu::Numerics::fast}) {
        for (int nkr : {17, 33}) {
            const MassGrid grid = make_mass_grid(nkr, 3.35e-14, 2.0);
            const KernelTableSet tables =
                build_tables(grid, default_pair_registry(), KernelParams{KernelFamily::golovin, 1.0, 1.5, 0.05});
            for (double cf : {0.0, 0.3, 1.0})
                for (std::uint64_t seed : {1ull, 42ull}) {
                    GridState s = make_synthetic_case({16, 8, 8, cf, seed, nkr, 3.35e-14, 2.0, 1e6});
                    char name[96];
                    std::snprintf(name, sizeof name, "liquid 16x8x8 nkr=%d cf=%.1f seed=%llu", nkr, cf,
                                  (unsigned long long)seed);
                    compare_case(name, s, tables, par3, 1.0, 1, nullptr, numerics);
                }
            GridState s = make_synthetic_case({12, 6, 10, 0.7, 5, nkr, 3.35e-14, 2.0, 1e6});
            fill_all_categories(s, 5);
            compare_case("all-category 12x6x10 substeps=3", s, tables, ser2, 1.5, 3, nullptr, numerics);
            const PatchTilePlan tiles = decompose(s.ranges, 2, 3);
            compare_case("all-category 12x6x10 2x3 tiles", s, tables, par3, 0.5, 1, &tiles, numerics);
        }
        // stiffness: coeff 1500 at dt 1 -> StiffnessError at the serial-first point
        const MassGrid grid = make_mass_grid(33, 3.35e-14, 2.0);
        const KernelTableSet stiff =
            build_tables(grid, default_pair_registry(), KernelParams{KernelFamily::golovin, 1500.0, 1.5, 0.0});
        GridState s = make_synthetic_case({6, 5, 7, 0.5, 11, 33, 3.35e-14, 2.0, 1e6});
        compare_case("stiffness (coeff 1500)", s, stiff, ser2, 1.0, 1, nullptr, numerics);
        const PatchTilePlan tiles = decompose(s.ranges, 3, 2);
        compare_case("stiffness with 3x2 tiles", s, stiff, par3, 1.0, 1, &tiles, numerics);
    }
    // argument errors: same exception types as the reference
    const MassGrid grid = make_mass_grid(33, 3.35e-14, 2.0);
    const KernelTableSet tables = build_tables(grid, default_pair_registry(), KernelParams{});
    GainTable gains(grid);
    GridState s = make_synthetic_case({4, 3, 5, 0.5, 3, 33, 3.35e-14, 2.0, 1e6});
    const PredicateMask mask = fission_predicates(s);
    StepContext ctx{&tables, &gains, CoalConfig{}, StubParams{0, 0}, nullptr, nullptr, nullptr, nullptr};
    auto both = [&](const char* name, const PredicateMask& m, const StepContext& c, const ExecPlan& p) {
        GridState a = s, b = s;
        const Outcome oa = run([&] { fissioned_step(a, m, c, p); });
        const Outcome ob = run([&] { gpu::fissioned_step(b, m, c, p); });
        CHECK(oa.type == ob.type && oa.type != "ok", "%s: reference %s vs gpu %s (%s)", name,
              oa.type.c_str(), ob.type.c_str(), ob.what.c_str());
        CHECK(bitwise_equal(b, s), "%s: gpu path touched the state", name);
        std::printf("  %-44s %-15s %s\n", name, ob.type.c_str(), ob.what.c_str());
    };
    both("collapse 3 + automatic scratch", mask, ctx,
         ExecPlan{StepMode::parallel, 3, 2, KernelStrategy::on_demand, ScratchStrategy::automatic});
    both("threads 0", mask, ctx, ExecPlan{StepMode::parallel, 2, 0, KernelStrategy::on_demand,
                                          ScratchStrategy::automatic});
    both("arena strategy without an arena", mask, ctx,
         ExecPlan{StepMode::serial, 2, 1, KernelStrategy::on_demand, ScratchStrategy::arena});
    PredicateMask stale = mask;
    stale.call_coal[3] ^= 1;
    both("stale mask", stale, ctx, ExecPlan{});
    PredicateMask wrong = mask;
    wrong.ranges.ide += 1;
    both("mask extents", wrong, ctx, ExecPlan{});
    StepContext noctx = ctx;
    noctx.gains = nullptr;
    both("no gain table", mask, noctx, ExecPlan{});
    gpu::release();
    if (g_fail) {
        std::printf("dropin FAILED (%d)\n", g_fail);
        return 1;
    }
    std::printf("dropin ok\n");
    return 0;
}
