// fsmoe/cost_models.hpp — alpha-beta duration models and their least-squares
// fit (drop-in for the reference's proj/src/include/fsmoe/cost_models.hpp).
// Communication kinds count 4-byte elements, gemm counts MACs.
#pragma once

#include <span>
#include <string>
#include <utility>
#include <vector>

#include "fsmoe/common.hpp"

namespace fsmoe {

struct LinearModel {
  double alpha_ms = 0.0;          // launch cost
  double beta_ms_per_unit = 0.0;  // per element / MAC
};

double predict_ms(const LinearModel& m, double n);              // alpha + n beta
double chunk_ms(const LinearModel& m, double n, int r);         // alpha + (n / r) beta, r >= 1
double invert_elements(const LinearModel& m, double t_ms);      // max(0, (t - alpha) / beta)

struct FitResult {
  LinearModel model;
  double r_squared = 0.0;
  bool clamped = false;
};

// OLS with non-negativity repair (alpha < 0: refit through the origin;
// beta < 0: constant model). Needs >= 2 samples.
FitResult fit_linear(std::span<const std::pair<double, double>> samples);

struct ClusterProfile {
  LinearModel a2a;
  LinearModel ag;
  LinearModel rs;
  LinearModel ar;
  LinearModel gemm;
};

struct BenchSample {
  std::string kind;  // a2a | ag | rs | ar | gemm
  double n = 0.0;
  double t_ms = 0.0;
};

struct ProfileFit {
  ClusterProfile profile;
  double min_r_squared = 0.0;
  std::vector<std::string> clamped_kinds;
};

// One model per kind; every kind required; FitQualityError below min_r2.
ProfileFit fit_profile(const std::vector<BenchSample>& samples, double min_r2);

}  // namespace fsmoe
