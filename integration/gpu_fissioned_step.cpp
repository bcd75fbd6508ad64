// gpu_fissioned_step.cpp -- coalbench::fissioned_step (driver.cpp:353-434) over the C ABI.
#include "gpu_fissioned_step.hpp"

#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "coalbench/errors.hpp"
#include "fsbm_coal.h"

namespace coalbench::gpu {

namespace {

struct Cache {
    Options opt;
    fsbm_ctx* ctx = nullptr;
    int device = -1;
    const KernelTableSet* tables = nullptr;
    std::vector<double> x, t750, t500; // what the device context was built from
    std::vector<int> abd;
    double ratio = 0.0;
};

Cache& cache() {
    static Cache c;
    return c;
}

std::mutex g_mu;

[[noreturn]] void rethrow(int status, const fsbm_error& e) {
    const std::string msg = fsbm_last_error();
    switch (status) {
    case FSBM_DOMAIN: throw DomainError(msg);
    case FSBM_SHAPE: throw ShapeError(msg);
    case FSBM_CONFIG: throw ConfigError(msg);
    case FSBM_STIFFNESS:
        if (e.has_point) throw StiffnessError(msg, e.category, e.bin, e.i, e.k, e.j);
        throw StiffnessError(msg, e.category, e.bin);
    case FSBM_ALLOC: throw AllocationError(msg, 0);
    default: throw Error("gpu fissioned_step: " + msg);
    }
}

/// The tables as the C ABI takes them (KernelTableSet layout [pair][i][j], kernels.hpp:105-107).
void snapshot_tables(const KernelTableSet& t, std::vector<double>& t750, std::vector<double>& t500,
                     std::vector<int>& abd) {
    const int n = t.nkr(), np = t.num_pairs();
    t750.resize(static_cast<std::size_t>(np) * n * n);
    t500.resize(t750.size());
    for (int p = 0; p < np; ++p)
        for (int i = 0; i < n; ++i) {
            std::memcpy(&t750[(static_cast<std::size_t>(p) * n + i) * n], t.row_750(p, i), n * sizeof(double));
            std::memcpy(&t500[(static_cast<std::size_t>(p) * n + i) * n], t.row_500(p, i), n * sizeof(double));
        }
    abd.clear();
    for (const auto& pr : t.pairs()) {
        abd.push_back(static_cast<int>(pr.source_a));
        abd.push_back(static_cast<int>(pr.source_b));
        abd.push_back(static_cast<int>(pr.dest));
    }
}

/// The cached context, rebuilt when the device, grid or table values change (the tables
/// are compared by value: KernelTableSet::mutable_750/500 allow edits after a first step).
fsbm_ctx* context_for(const GridState& state, const KernelTableSet& tables) {
    Cache& c = cache();
    std::vector<double> t750, t500;
    std::vector<int> abd;
    snapshot_tables(tables, t750, t500, abd);
    if (c.ctx && c.device == c.opt.device && c.tables == &tables && c.x == state.grid.x &&
        c.ratio == state.grid.ratio && c.t750 == t750 && c.t500 == t500 && c.abd == abd)
        return c.ctx;
    if (c.ctx) fsbm_ctx_destroy(c.ctx);
    c.ctx = nullptr;
    fsbm_ctx* ctx = nullptr;
    const int st = fsbm_ctx_create(c.opt.device, state.nkr(), state.grid.x.data(), state.grid.ratio,
                                   tables.num_pairs(), abd.data(), t750.data(), t500.data(), &ctx);
    if (st != FSBM_OK) rethrow(st, fsbm_error{});
    c.ctx = ctx;
    c.device = c.opt.device;
    c.tables = &tables;
    c.x = state.grid.x;
    c.ratio = state.grid.ratio;
    c.t750.swap(t750);
    c.t500.swap(t500);
    c.abd.swap(abd);
    return ctx;
}

} // namespace

void set_options(const Options& o) {
    std::lock_guard<std::mutex> lk(g_mu);
    cache().opt = o;
}

Options options() {
    std::lock_guard<std::mutex> lk(g_mu);
    return cache().opt;
}

void release() {
    std::lock_guard<std::mutex> lk(g_mu);
    Cache& c = cache();
    if (c.ctx) fsbm_ctx_destroy(c.ctx);
    c.ctx = nullptr;
    c.tables = nullptr;
}

void fissioned_step(GridState& state, const PredicateMask& mask, const StepContext& ctx,
                    const ExecPlan& plan) {
    using Clock = std::chrono::steady_clock;
    const auto t0 = Clock::now();
    std::lock_guard<std::mutex> lk(g_mu);
    // the reference's checks, in its order (driver.cpp:355-367); the stale-mask scan and
    // the plan rules are repeated by the library with the same messages
    validate_plan(plan);
    if (ctx.tables == nullptr || ctx.gains == nullptr)
        throw DomainError("fissioned_step: context must supply tables and gains");
    if (plan.scratch_strategy == ScratchStrategy::arena) { // check_arena (driver.cpp:122-130)
        if (ctx.arena == nullptr)
            throw ConfigError("step: arena scratch strategy requires an allocated arena");
        if (ctx.arena->ni() != state.ranges.ni() || ctx.arena->nk() != state.ranges.nk() ||
            ctx.arena->nj() != state.ranges.nj() || ctx.arena->nkr() != state.nkr())
            throw ShapeError("step: arena extents do not match the state");
    }
    if (!(mask.ranges == state.ranges))
        throw ShapeError("fissioned_step: mask extents do not match the state");
    const std::size_t np = state.ranges.npoints();
    const std::size_t nkr = static_cast<std::size_t>(state.nkr());
    if (state.temperature.size() != np || state.pressure.size() != np ||
        mask.call_coal.size() != np)
        throw ShapeError("fissioned_step: state/mask arrays do not match the ranges");
    for (int c = 0; c < kNumCategories; ++c)
        if (state.bins[c].size() != np * nkr)
            throw ShapeError("coal_step: state distribution size does not match nkr");
    if (ctx.tables->nkr() != state.nkr() || ctx.gains->nkr() != state.nkr())
        throw ShapeError("coal_step: grid, tables and gain table disagree on nkr");

    fsbm_ctx* dctx = context_for(state, *ctx.tables);
    const Ranges& r = state.ranges;
    const fsbm_ranges fr{r.ids, r.ide, r.kds, r.kde, r.jds, r.jde};
    const fsbm_plan fp{plan.mode == StepMode::parallel ? 1 : 0, plan.collapse, plan.threads,
                       plan.kernel_strategy == KernelStrategy::precomputed ? FSBM_PRECOMPUTED
                                                                           : FSBM_ON_DEMAND,
                       plan.scratch_strategy == ScratchStrategy::arena ? FSBM_ARENA : FSBM_AUTOMATIC,
                       cache().opt.numerics == Numerics::exact ? FSBM_NUMERICS_EXACT
                                                               : FSBM_NUMERICS_FAST};
    std::vector<fsbm_tile> tiles; // patch-major, tile-minor: run order of driver.cpp:394-425
    if (ctx.tiles != nullptr)
        for (const auto& patch : ctx.tiles->patches)
            for (const auto& t : patch.tiles) tiles.push_back(fsbm_tile{t.its, t.ite, t.jts, t.jte});
    double* bins[FSBM_NCAT];
    for (int c = 0; c < kNumCategories; ++c) bins[c] = state.bins[c].data();
    fsbm_counters cnt{0, 0, 0};
    fsbm_error err{-1, -1, 0, 0, 0, 0, 0.0};
    const auto t1 = Clock::now();
    const int st = fsbm_step_grid_host(dctx, fr, bins, state.pressure.data(),
                                       state.temperature.data(), mask.call_coal.data(),
                                       ctx.coal.dt, ctx.coal.substeps, &fp,
                                       tiles.empty() ? nullptr : tiles.data(),
                                       static_cast<int>(tiles.size()), &cnt, &err);
    const auto t2 = Clock::now();
    if (st == FSBM_OK || st == FSBM_STIFFNESS) { // the reference counts work up to the throw
        if (ctx.counters != nullptr) {
            ctx.counters->coal.triples.fetch_add(cnt.triples, std::memory_order_relaxed);
            ctx.counters->coal.points.fetch_add(cnt.points, std::memory_order_relaxed);
        }
        ctx.tables->add_evals(cnt.kernel_evals);
    }
    if (ctx.timings != nullptr) {
        ctx.timings->coal_s += std::chrono::duration<double>(t2 - t1).count();
        ctx.timings->step_s += std::chrono::duration<double>(t2 - t0).count();
    }
    if (st != FSBM_OK) rethrow(st, err);
}

} // namespace coalbench::gpu
