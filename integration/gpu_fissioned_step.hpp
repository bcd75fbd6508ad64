// gpu_fissioned_step.hpp -- the C++ drop-in for coalbench::fissioned_step on a B200.
//
// Same signature and exception contract as the reference's
//   void fissioned_step(GridState&, const PredicateMask&, const StepContext&, const ExecPlan&)
// (proj/include/coalbench/driver.hpp:179-180, proj/src/driver.cpp:353-434); phase 2
// (coal_step at every mask-true point, coalescence.cpp:204-339) runs in the sm_100a kernels
// of libfsbm_coal.so through its C ABI (include/fsbm_coal.h).  Errors are rethrown as the
// reference's coalbench::ConfigError / ShapeError / DomainError / StiffnessError (with
// at_point coordinates) / AllocationError (errors.hpp:10-74).
//
// Phase 1 of the reference step (stub_rows: nucleation/condensation stand-in spins that
// write no state, driver.cpp:139-168) is not part of the hot path; a maintainer who wants
// its counters keeps it in driver.cpp and calls this function for phase 2.
#pragma once

#include "coalbench/driver.hpp"

namespace coalbench::gpu {

enum class Numerics {
    fast,  ///< FP64 tensor-core kernels; per bin within 1e-12 of coal_step
    exact, ///< bitwise identical to coal_step (reference operation order, no FMA)
};

struct Options {
    int device = 0;
    Numerics numerics = Numerics::fast;
};

/// Process-wide options for subsequent calls (not thread-safe against concurrent steps).
void set_options(const Options& options);
Options options();

/// Drop-in for coalbench::fissioned_step.  The device context (tables, registry, gain
/// table) is built on first use and rebuilt when the table set or grid changes.
void fissioned_step(GridState& state, const PredicateMask& mask, const StepContext& ctx,
                    const ExecPlan& plan);

/// Releases the cached device context.
void release();

} // namespace coalbench::gpu
