// ref_wrap.cpp — TEST INFRASTRUCTURE ONLY.
//
// C-array wrapper around the reference library compiled from its own sources
// under /root/reference/proj/src (see oracle/Makefile). The Makefile compiles
// every TU, this one included, with -Dfsmoe=fsmoe_ref so the reference's
// symbols live in namespace fsmoe_ref and can never collide with the product
// library's fsmoe:: symbols. Nothing here re-implements reference logic: it
// only marshals flat arrays into the reference types and back.
//
// Used by oracle/gen_golden.py (golden fixtures), tests (when the build
// exists) and bench.py --impl reference (CPU baseline).
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "fsmoe/common.hpp"
#include "fsmoe/cost_models.hpp"
#include "fsmoe/grad_partition.hpp"
#include "fsmoe/pipeline_optimizer.hpp"
#include "fsmoe/schedule_sim.hpp"
#include "fsmoe/workload.hpp"

namespace {

using namespace fsmoe;  // renamed to fsmoe_ref by the build

void put_err(char* err, int errlen, const char* what) {
  if (err && errlen > 0) {
    std::strncpy(err, what, static_cast<size_t>(errlen) - 1);
    err[errlen - 1] = '\0';
  }
}

template <class F>
int guarded(char* err, int errlen, F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    put_err(err, errlen, e.what());
    return exit_config_error;
  } catch (const FitQualityError& e) {
    put_err(err, errlen, e.what());
    return exit_fit_quality;
  } catch (const InvariantError& e) {
    put_err(err, errlen, e.what());
    return exit_invariant;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

Matrix make_matrix(int rows, int cols, const double* data) {
  Matrix m;
  m.rows = rows;
  m.cols = cols;
  size_t n = static_cast<size_t>(rows > 0 ? rows : 0) * static_cast<size_t>(cols > 0 ? cols : 0);
  m.v.assign(n, 0.0);
  if (data && n) std::memcpy(m.v.data(), data, n * sizeof(double));
  return m;
}

LayerConfig make_layer(const int* ints, const double* dbls) {
  // ints: batch heads seq_len model_dim hidden_scale unlimited ffn experts top_k
  //       has_override
  // dbls: capacity_factor t_olp_dense_ms grad_override
  LayerConfig c;
  c.batch = ints[0];
  c.heads = ints[1];
  c.seq_len = ints[2];
  c.model_dim = ints[3];
  c.hidden_scale = ints[4];
  c.unlimited_capacity = ints[5] != 0;
  c.ffn = ints[6] ? LayerConfig::Ffn::gated3 : LayerConfig::Ffn::simple;
  c.experts = ints[7];
  c.top_k = ints[8];
  c.capacity_factor = dbls[0];
  c.t_olp_dense_ms = dbls[1];
  if (ints[9]) c.grad_elements_override = dbls[2];
  return c;
}

ClusterProfile make_profile(const double* p) {
  ClusterProfile c;
  c.a2a = {p[0], p[1]};
  c.ag = {p[2], p[3]};
  c.rs = {p[4], p[5]};
  c.ar = {p[6], p[7]};
  c.gemm = {p[8], p[9]};
  return c;
}

void put_profile(const ClusterProfile& c, double* p) {
  const LinearModel* ms[5] = {&c.a2a, &c.ag, &c.rs, &c.ar, &c.gemm};
  for (int i = 0; i < 5; ++i) {
    p[2 * i] = ms[i]->alpha_ms;
    p[2 * i + 1] = ms[i]->beta_ms_per_unit;
  }
}

TaskVolumes make_volumes(const double* v) {
  // a2a ag rs gemm_macs gemm_count grad capacity
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

int ref_run_gate(int kind, int top_k, uint64_t seed, int tokens, int dim,
                 const double* x, int ws_rows, int ws_cols, const double* w_score,
                 int wn_rows, int wn_cols, const double* w_noise, int pj_rows,
                 int pj_cols, const double* proj, int* pick_token,
                 int* pick_expert, double* pick_weight, long long* n_picks,
                 char* err, int errlen) {
  *n_picks = 0;
  return guarded(err, errlen, [&] {
    GateParams params;
    params.score_weights = make_matrix(ws_rows, ws_cols, w_score);
    params.noise_weights = make_matrix(wn_rows, wn_cols, w_noise);
    params.projection = make_matrix(pj_rows, pj_cols, proj);
    GateConfig g;
    g.kind = static_cast<GateKind>(kind);
    g.top_k = top_k;
    g.seed = seed;
    GateOutput out = run_gate(make_matrix(tokens, dim, x), g, params);
    for (size_t i = 0; i < out.picks.size(); ++i) {
      pick_token[i] = out.picks[i].token;
      pick_expert[i] = out.picks[i].expert;
      pick_weight[i] = out.picks[i].weight;
    }
    *n_picks = static_cast<long long>(out.picks.size());
  });
}

int ref_dispatch(int tokens, int dim, const double* x, int experts,
                 long long n_picks, const int* pick_token, const int* pick_expert,
                 long long capacity, double* buffers, int* slot_of_pick,
                 long long* fill, long long* dropped, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    GateOutput g;
    g.tokens = tokens;
    g.experts = experts;
    g.picks.resize(static_cast<size_t>(n_picks));
    for (long long i = 0; i < n_picks; ++i)
      g.picks[i] = {pick_token[i], pick_expert[i], 0.0};
    DispatchResult d = dispatch_tokens(make_matrix(tokens, dim, x), g, capacity);
    std::memcpy(buffers, d.buffers.v.data(), d.buffers.v.size() * sizeof(double));
    for (size_t i = 0; i < d.slot_of_pick.size(); ++i) slot_of_pick[i] = d.slot_of_pick[i];
    for (size_t e = 0; e < d.fill.size(); ++e) fill[e] = d.fill[e];
    *dropped = d.dropped;
  });
}

int ref_combine(int buf_rows, int buf_cols, const double* buffers, int tokens,
                int experts, long long n_picks, const int* pick_token,
                const int* pick_expert, const double* pick_weight,
                long long n_slots, const int* slot_of_pick, int model_dim,
                double* y, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    GateOutput g;
    g.tokens = tokens;
    g.experts = experts;
    g.picks.resize(static_cast<size_t>(n_picks));
    for (long long i = 0; i < n_picks; ++i)
      g.picks[i] = {pick_token[i], pick_expert[i], pick_weight[i]};
    DispatchResult d;
    d.experts = experts;
    d.slot_of_pick.assign(slot_of_pick, slot_of_pick + n_slots);
    Matrix out = combine_tokens(make_matrix(buf_rows, buf_cols, buffers), g, d, model_dim);
    std::memcpy(y, out.v.data(), out.v.size() * sizeof(double));
  });
}

long long ref_capacity_tokens(const int* ints, const double* dbls, char* err, int errlen) {
  long long cap = -1;
  int rc = guarded(err, errlen, [&] { cap = capacity_tokens(make_layer(ints, dbls)); });
  return rc ? -1 : cap;
}

// pints: total_gpus gpus_per_node data_parallel tensor_parallel expert_parallel expert_shard
// out:   a2a ag rs gemm_macs gemm_count grad capacity
int ref_derive_volumes(const int* ints, const double* dbls, const int* pints,
                       double* out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    ParallelConfig p;
    p.total_gpus = pints[0];
    p.gpus_per_node = pints[1];
    p.data_parallel = pints[2];
    p.tensor_parallel = pints[3];
    p.expert_parallel = pints[4];
    p.expert_shard = pints[5];
    TaskVolumes v = derive_volumes(make_layer(ints, dbls), p);
    out[0] = v.a2a_elements;
    out[1] = v.ag_elements;
    out[2] = v.rs_elements;
    out[3] = v.gemm_macs;
    out[4] = v.gemm_count;
    out[5] = v.grad_elements;
    out[6] = static_cast<double>(v.capacity);
  });
}

// ---- control plane -------------------------------------------------------

// kinds: 0 a2a 1 ag 2 rs 3 ar 4 gemm ; out_profile: 10 doubles ; out_meta:
// [min_r2, clamped_mask]
int ref_fit_profile(int n, const int* kinds, const double* ns, const double* ts,
                    double min_r2, double* out_profile, double* out_meta,
                    char* err, int errlen) {
  static const char* names[5] = {"a2a", "ag", "rs", "ar", "gemm"};
  return guarded(err, errlen, [&] {
    std::vector<BenchSample> s(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      s[i].kind = (kinds[i] >= 0 && kinds[i] < 5) ? names[kinds[i]] : "bogus";
      s[i].n = ns[i];
      s[i].t_ms = ts[i];
    }
    ProfileFit f = fit_profile(s, min_r2);
    put_profile(f.profile, out_profile);
    out_meta[0] = f.min_r_squared;
    double mask = 0;
    for (auto& k : f.clamped_kinds)
      for (int j = 0; j < 5; ++j)
        if (k == names[j]) mask += double(1 << j);
    out_meta[1] = mask;
  });
}

// out: [r, case, t_moe, q0..q6, boundary]
int ref_find_degree(const double* vol, const double* prof, double t_gar,
                    int exp_mult, int r_max, double* out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    PhaseInputs in;
    in.volumes = make_volumes(vol);
    in.profile = make_profile(prof);
    in.t_gar_ms = t_gar;
    in.exp_multiplier = exp_mult;
    DegreeChoice c = find_optimal_pipeline_degree(in, r_max);
    out[0] = c.r;
    out[1] = c.case_id;
    out[2] = c.t_moe_ms;
    for (int i = 0; i < 7; ++i) out[3 + i] = c.q[i] ? 1.0 : 0.0;
    out[10] = c.boundary ? 1.0 : 0.0;
  });
}

// out: r_fwd case_fwd t_fwd boundary_fwd r_bwd case_bwd t_bwd boundary_bwd
//      t_gar_bwd t_olp_moe_bwd
int ref_plan_layer(const double* vol, const double* prof, double t_gar_bwd,
                   int r_max, double* out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    PipelinePlan p = plan_layer(make_volumes(vol), make_profile(prof), t_gar_bwd, r_max);
    out[0] = p.r_fwd;
    out[1] = p.case_fwd;
    out[2] = p.t_moe_fwd_ms;
    out[3] = p.boundary_fwd;
    out[4] = p.r_bwd;
    out[5] = p.case_bwd;
    out[6] = p.t_moe_bwd_ms;
    out[7] = p.boundary_bwd;
    out[8] = p.t_gar_bwd_ms;
    out[9] = p.t_olp_moe_bwd_ms;
  });
}

// layers: n x (7 volume doubles, t_olp_dense, n_grad)
// de: population generations weight crossover seed
// out per layer: n_first n_first_dense n_first_moe x_g t_gar degree case
//                t_olp_moe t_olp_dense ; then tail_elements tail_ms objective step2_ran
int ref_build_partition_plan(int n, const double* layers, const double* prof,
                             const double* de, int r_max, double* out,
                             char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<GradLayer> ls(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      ls[i].volumes = make_volumes(layers + 9 * i);
      ls[i].t_olp_dense_ms = layers[9 * i + 7];
      ls[i].n_grad = layers[9 * i + 8];
    }
    DeParams d;
    d.population = static_cast<int>(de[0]);
    d.generations = static_cast<int>(de[1]);
    d.weight = de[2];
    d.crossover = de[3];
    d.seed = static_cast<std::uint64_t>(de[4]);
    PartitionPlan p = build_partition_plan(ls, make_profile(prof), d, r_max);
    for (int i = 0; i < n; ++i) {
      const auto& a = p.layers[i];
      double* o = out + 9 * i;
      o[0] = a.n_first;
      o[1] = a.n_first_dense;
      o[2] = a.n_first_moe;
      o[3] = a.x_g;
      o[4] = a.t_gar_ms;
      o[5] = a.window.degree;
      o[6] = a.window.case_id;
      o[7] = a.window.t_olp_moe_ms;
      o[8] = a.window.t_olp_dense_ms;
    }
    out[9 * n + 0] = p.tail_elements;
    out[9 * n + 1] = p.tail_ms;
    out[9 * n + 2] = p.objective_ms;
    out[9 * n + 3] = p.step2_ran ? 1.0 : 0.0;
  });
}

// Simulates the chosen style for a stage built from volumes; out:
// [makespan, busy0, busy1, busy2, n_tasks] then per task (start, end).
int ref_simulate_stage(const double* vol, const double* prof, int exp_mult,
                       int r, int n_sync, const double* sync_ms, int style,
                       double* out, int out_cap, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<double> gs(sync_ms, sync_ms + n_sync);
    StageTimes st = stage_times(make_volumes(vol), make_profile(prof), exp_mult, r, gs);
    Dag dag = build_baseline_dag(static_cast<ScheduleStyle>(style), st);
    Timeline tl = simulate(dag);
    out[0] = tl.makespan_ms;
    out[1] = tl.busy_ms[0];
    out[2] = tl.busy_ms[1];
    out[3] = tl.busy_ms[2];
    out[4] = static_cast<double>(tl.tasks.size());
    for (size_t i = 0; i < tl.tasks.size() && 5 + 2 * i + 1 < static_cast<size_t>(out_cap); ++i) {
      out[5 + 2 * i] = tl.tasks[i].start_ms;
      out[6 + 2 * i] = tl.tasks[i].end_ms;
    }
  });
}

int ref_brute_force_degree(const double* vol, const double* prof, double t_gar,
                           int exp_mult, int r_max, double* out, char* err,
                           int errlen) {
  return guarded(err, errlen, [&] {
    BruteForceResult b = brute_force_best_degree(make_volumes(vol), make_profile(prof),
                                                 t_gar, exp_mult, r_max);
    out[0] = b.r;
    out[1] = b.makespan_ms;
  });
}

}  // extern "C"
