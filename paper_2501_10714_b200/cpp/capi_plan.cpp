// capi_plan.cpp — extern "C" surface of the host control plane
// (include/fsmoe_plan.h). Same flat-array conventions as the test wrapper of
// the reference (oracle/ref_wrap.cpp) so the two are compared call for call.
#include <algorithm>
#include <cstdint>
#include <exception>
#include <string>
#include <vector>

#include "fsmoe/common.hpp"
#include "fsmoe/cost_models.hpp"
#include "fsmoe/grad_partition.hpp"
#include "fsmoe/pipeline_optimizer.hpp"
#include "fsmoe/schedule_sim.hpp"
#include "fsmoe/workload.hpp"
#include "fsmoe_plan.h"

extern "C" const char* fsmoe_layer_last_error(void);

namespace fsmoe {
void set_layer_error(const std::string& msg);  // capi_layer.cpp
}

namespace {

using namespace fsmoe;

template <class F>
int run(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    set_layer_error(e.what());
    return exit_config_error;
  } catch (const FitQualityError& e) {
    set_layer_error(e.what());
    return exit_fit_quality;
  } catch (const InvariantError& e) {
    set_layer_error(e.what());
    return exit_invariant;
  } catch (const std::exception& e) {
    set_layer_error(e.what());
    return 1;
  }
}

LayerConfig layer_of(const int* i, const double* d) {
  LayerConfig c;
  c.batch = i[0];
  c.heads = i[1];
  c.seq_len = i[2];
  c.model_dim = i[3];
  c.hidden_scale = i[4];
  c.unlimited_capacity = i[5] != 0;
  c.ffn = i[6] ? LayerConfig::Ffn::gated3 : LayerConfig::Ffn::simple;
  c.experts = i[7];
  c.top_k = i[8];
  c.capacity_factor = d[0];
  c.t_olp_dense_ms = d[1];
  if (i[9]) c.grad_elements_override = d[2];
  return c;
}

ClusterProfile profile_of(const double* p) {
  ClusterProfile c;
  LinearModel* m[5] = {&c.a2a, &c.ag, &c.rs, &c.ar, &c.gemm};
  for (int k = 0; k < 5; ++k) *m[k] = {p[2 * k], p[2 * k + 1]};
  return c;
}

TaskVolumes volumes_of(const double* v) {
  TaskVolumes t;
  t.a2a_elements = v[0];
  t.ag_elements = v[1];
  t.rs_elements = v[2];
  t.gemm_macs = v[3];
  t.gemm_count = static_cast<int>(v[4]);
  t.grad_elements = v[5];
  t.capacity = static_cast<long long>(v[6]);
  return t;
}

}  // namespace

extern "C" {

long long fsmoe_capacity_tokens(const int* li, const double* ld) {
  long long cap = -1;
  if (run([&] { cap = capacity_tokens(layer_of(li, ld)); })) return -1;
  return cap;
}

int fsmoe_derive_volumes(const int* li, const double* ld, const int* p, double* out) {
  return run([&] {
    ParallelConfig pc{p[0], p[1], p[2], p[3], p[4], p[5]};
    const TaskVolumes v = derive_volumes(layer_of(li, ld), pc);
    const double vals[7] = {v.a2a_elements, v.ag_elements, v.rs_elements, v.gemm_macs,
                            static_cast<double>(v.gemm_count), v.grad_elements,
                            static_cast<double>(v.capacity)};
    std::copy(vals, vals + 7, out);
  });
}

int fsmoe_pipeline_chunks(long long C, int r, int* out) {
  // mirrors make_chunks() of moe_layer.cpp
  const long long ng = (C + 127) / 128;
  if (r < 1) r = 1;
  if (r > ng) r = static_cast<int>(ng);
  for (int i = 0; i < r; ++i) {
    out[2 * i] = static_cast<int>((i * ng) / r * 128);
    out[2 * i + 1] = static_cast<int>(std::min(((i + 1) * ng) / r * 128, C));
  }
  return r;
}

int fsmoe_fit_profile(int n, const int* kinds, const double* ns, const double* ts, double min_r2,
                      double* prof, double* meta) {
  static const char* names[5] = {"a2a", "ag", "rs", "ar", "gemm"};
  return run([&] {
    std::vector<BenchSample> s(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) s[i] = {kinds[i] >= 0 && kinds[i] < 5 ? names[kinds[i]] : "bogus", ns[i], ts[i]};
    const ProfileFit f = fit_profile(s, min_r2);
    const LinearModel* m[5] = {&f.profile.a2a, &f.profile.ag, &f.profile.rs, &f.profile.ar, &f.profile.gemm};
    for (int k = 0; k < 5; ++k) {
      prof[2 * k] = m[k]->alpha_ms;
      prof[2 * k + 1] = m[k]->beta_ms_per_unit;
    }
    meta[0] = f.min_r_squared;
    double mask = 0;
    for (const auto& k : f.clamped_kinds)
      for (int j = 0; j < 5; ++j)
        if (k == names[j]) mask += double(1 << j);
    meta[1] = mask;
  });
}

int fsmoe_find_degree(const double* vol, const double* prof, double t_gar, int mult, int r_max,
                      double* out) {
  return run([&] {
    const DegreeChoice c =
        find_optimal_pipeline_degree(PhaseInputs{volumes_of(vol), profile_of(prof), t_gar, mult}, r_max);
    out[0] = c.r;
    out[1] = c.case_id;
    out[2] = c.t_moe_ms;
    for (int i = 0; i < 7; ++i) out[3 + i] = c.q[i] ? 1.0 : 0.0;
    out[10] = c.boundary ? 1.0 : 0.0;
  });
}

int fsmoe_plan_layer(const double* vol, const double* prof, double t_gar_bwd, int r_max, double* out) {
  return run([&] {
    const PipelinePlan p = plan_layer(volumes_of(vol), profile_of(prof), t_gar_bwd, r_max);
    const double vals[10] = {double(p.r_fwd), double(p.case_fwd), p.t_moe_fwd_ms, double(p.boundary_fwd),
                             double(p.r_bwd), double(p.case_bwd), p.t_moe_bwd_ms, double(p.boundary_bwd),
                             p.t_gar_bwd_ms, p.t_olp_moe_bwd_ms};
    std::copy(vals, vals + 10, out);
  });
}

int fsmoe_build_partition_plan(int n, const double* layers, const double* prof, const double* de,
                               int r_max, double* out) {
  return run([&] {
    std::vector<GradLayer> ls(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      ls[i].volumes = volumes_of(layers + 9 * i);
      ls[i].t_olp_dense_ms = layers[9 * i + 7];
      ls[i].n_grad = layers[9 * i + 8];
    }
    DeParams d;
    d.population = static_cast<int>(de[0]);
    d.generations = static_cast<int>(de[1]);
    d.weight = de[2];
    d.crossover = de[3];
    d.seed = static_cast<std::uint64_t>(de[4]);
    const PartitionPlan p = build_partition_plan(ls, profile_of(prof), d, r_max);
    for (int i = 0; i < n; ++i) {
      const LayerAssignment& a = p.layers[i];
      const double vals[9] = {a.n_first, a.n_first_dense, a.n_first_moe, a.x_g, a.t_gar_ms,
                              double(a.window.degree), double(a.window.case_id),
                              a.window.t_olp_moe_ms, a.window.t_olp_dense_ms};
      std::copy(vals, vals + 9, out + 9 * i);
    }
    out[9 * n + 0] = p.tail_elements;
    out[9 * n + 1] = p.tail_ms;
    out[9 * n + 2] = p.objective_ms;
    out[9 * n + 3] = p.step2_ran ? 1.0 : 0.0;
  });
}

int fsmoe_simulate_stage(const double* vol, const double* prof, int mult, int r, int n_sync,
                         const double* sync_ms, int style, double* out, int out_cap) {
  return run([&] {
    if (style < 0 || style > 3) throw ConfigError("unknown schedule style");
    const StageTimes st = stage_times(volumes_of(vol), profile_of(prof), mult, r,
                                      std::vector<double>(sync_ms, sync_ms + n_sync));
    const Dag dag = build_baseline_dag(static_cast<ScheduleStyle>(style), st);
    const Timeline tl = simulate(dag);
    out[0] = tl.makespan_ms;
    out[1] = tl.busy_ms[0];
    out[2] = tl.busy_ms[1];
    out[3] = tl.busy_ms[2];
    out[4] = static_cast<double>(tl.tasks.size());
    for (size_t i = 0; i < tl.tasks.size() && 6 + 2 * i < static_cast<size_t>(out_cap); ++i) {
      out[5 + 2 * i] = tl.tasks[i].start_ms;
      out[6 + 2 * i] = tl.tasks[i].end_ms;
    }
  });
}

int fsmoe_brute_force_degree(const double* vol, const double* prof, double t_gar, int mult,
                             int r_max, double* out) {
  return run([&] {
    const BruteForceResult b = brute_force_best_degree(volumes_of(vol), profile_of(prof), t_gar, mult, r_max);
    out[0] = b.r;
    out[1] = b.makespan_ms;
  });
}

}  // extern "C"
