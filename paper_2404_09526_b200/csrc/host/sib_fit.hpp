// Cost-model fitting for the measured-SIB loop: B200-measured
// prefill and decode times become the coefficients of the reference's
// scaling information base, so the unchanged scheduler plans with them.
#pragma once

#include <array>
#include <cstddef>

namespace esp {

// Least squares y ~ c0 + c1*x1 + c2*x2 with the reference's admissibility
// rule (fit_prefill_coefficients, cost_model.cpp:86-135): columns scaled to
// unit norm, solved by column-pivoted QR over the active columns
// (solve_active, cost_model.cpp:36-50, rank tolerance 1e-9), the most
// negative coefficient dropped and the rest refitted until all are >= 0.
// Fewer than three samples or a rank-deficient active design throw
// ConfigError (the reference's UnderdeterminedError).
//   prefill: x1 = sum of lengths, x2 = sum of squared lengths (cost_model.cpp:169-173)
//   decode : x1 = batch (/ masters above the compute-bound threshold),
//            x2 = resident KV / dop (cost_model.cpp:175-187)
std::array<double, 3> fit_cost(const double* x1, const double* x2, const double* y, size_t n);

}  // namespace esp
