// planner.cpp — the FSMoE control plane that configures the B200 executor,
// restated from the reference's cost_models.cpp, schedule_sim.cpp,
// pipeline_optimizer.cpp and grad_partition.cpp (proj/src). It runs once per
// layer shape on the host, so it stays plain C++; its
// outputs (r_fwd, r_bwd, allreduce slices) must equal the reference's for the
// same profile, so every formula keeps the reference's evaluation order
// (tests/test_planner.py compares against the reference compiled from its
// sources).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <deque>
#include <map>
#include <random>
#include <string>

#include "fsmoe/cost_models.hpp"
#include "fsmoe/grad_partition.hpp"
#include "fsmoe/pipeline_optimizer.hpp"
#include "fsmoe/schedule_sim.hpp"

namespace fsmoe {

// ============================================================ cost models ==
// (cost_models.cpp:9-125)

double predict_ms(const LinearModel& m, double n) { return m.alpha_ms + n * m.beta_ms_per_unit; }

double chunk_ms(const LinearModel& m, double n, int r) {
  if (r < 1) throw ConfigError("chunk_ms: degree must be >= 1");
  return m.alpha_ms + (n / r) * m.beta_ms_per_unit;
}

double invert_elements(const LinearModel& m, double t_ms) {
  if (m.beta_ms_per_unit <= 0.0) throw ConfigError("invert_elements: beta must be positive");
  return std::max(0.0, (t_ms - m.alpha_ms) / m.beta_ms_per_unit);
}

namespace {

double coefficient_of_determination(std::span<const std::pair<double, double>> pts,
                                    const LinearModel& m) {
  double mean = 0;
  for (const auto& p : pts) mean += p.second;
  mean /= static_cast<double>(pts.size());
  double res = 0, tot = 0;
  for (const auto& p : pts) {
    const double err = p.second - predict_ms(m, p.first);
    res += err * err;
    const double dev = p.second - mean;
    tot += dev * dev;
  }
  if (tot == 0.0) return res == 0.0 ? 1.0 : 0.0;
  return 1.0 - res / tot;
}

constexpr const char* kKinds[5] = {"a2a", "ag", "rs", "ar", "gemm"};

}  // namespace

FitResult fit_linear(std::span<const std::pair<double, double>> pts) {
  if (pts.size() < 2) throw ConfigError("fit_linear: need at least 2 samples");
  double n = static_cast<double>(pts.size()), sx = 0, sy = 0, sxx = 0, sxy = 0;
  for (const auto& [xv, yv] : pts) {
    sx += xv;
    sy += yv;
    sxx += xv * xv;
    sxy += xv * yv;
  }
  FitResult f;
  const double det = n * sxx - sx * sx;
  if (det == 0.0) {
    f.model = {sy / n, 0.0};  // slope unidentifiable: constant model
  } else {
    f.model.beta_ms_per_unit = (n * sxy - sx * sy) / det;
    f.model.alpha_ms = (sy - f.model.beta_ms_per_unit * sx) / n;
  }
  if (f.model.alpha_ms < 0.0) {  // through the origin
    f.model = {0.0, sxx > 0.0 ? sxy / sxx : 0.0};
    f.clamped = true;
  }
  if (f.model.beta_ms_per_unit < 0.0) {  // constant
    f.model = {sy / n, 0.0};
    f.clamped = true;
  }
  f.r_squared = coefficient_of_determination(pts, f.model);
  return f;
}

ProfileFit fit_profile(const std::vector<BenchSample>& samples, double min_r2) {
  std::map<std::string, std::vector<std::pair<double, double>>> groups;
  for (const auto& s : samples) groups[s.kind].emplace_back(s.n, s.t_ms);
  for (const char* k : kKinds)
    if (!groups.count(k))
      throw ConfigError(std::string("fit_profile: no samples for kind '") + k + "'");
  for (const auto& g : groups)
    if (std::find_if(std::begin(kKinds), std::end(kKinds),
                     [&](const char* k) { return g.first == k; }) == std::end(kKinds))
      throw ConfigError("fit_profile: unknown kind '" + g.first + "'");
  ProfileFit out;
  out.min_r_squared = 1.0;
  LinearModel* dst[5] = {&out.profile.a2a, &out.profile.ag, &out.profile.rs, &out.profile.ar,
                         &out.profile.gemm};
  for (int i = 0; i < 5; ++i) {
    const FitResult f = fit_linear(groups[kKinds[i]]);
    *dst[i] = f.model;
    out.min_r_squared = std::min(out.min_r_squared, f.r_squared);
    if (f.clamped) out.clamped_kinds.push_back(kKinds[i]);
    if (f.r_squared < min_r2)
      throw FitQualityError(std::string("fit_profile: kind '") + kKinds[i] + "' r^2 " +
                            std::to_string(f.r_squared) + " below threshold " +
                            std::to_string(min_r2));
  }
  return out;
}

// ========================================================= schedule sim ==
// (schedule_sim.cpp:12-434)

Resource resource_of(OpKind kind) {
  switch (kind) {
    case OpKind::a2a_dispatch:
    case OpKind::a2a_combine:
    case OpKind::grad_allreduce: return Resource::inter_link;
    case OpKind::allgather:
    case OpKind::reducescatter: return Resource::intra_link;
    case OpKind::expert:
    case OpKind::dense_compute: return Resource::compute;
  }
  return Resource::compute;
}

const char* to_string(OpKind kind) {
  static const char* names[] = {"a2a_dispatch", "allgather",      "expert",       "reducescatter",
                                "a2a_combine",  "grad_allreduce", "dense_compute"};
  const int i = static_cast<int>(kind);
  return i >= 0 && i < 7 ? names[i] : "?";
}

const char* to_string(Resource res) {
  static const char* names[] = {"inter", "intra", "compute"};
  const int i = static_cast<int>(res);
  return i >= 0 && i < 3 ? names[i] : "?";
}

ScheduleStyle style_from_string(const std::string& s) {
  static const std::pair<const char*, ScheduleStyle> table[] = {
      {"fsmoe", ScheduleStyle::fsmoe},
      {"fsmoe_no_iio", ScheduleStyle::fsmoe_no_iio},
      {"pipemoe", ScheduleStyle::pipemoe},
      {"sequential", ScheduleStyle::sequential}};
  for (const auto& [name, style] : table)
    if (s == name) return style;
  throw ConfigError("unknown schedule style '" + s + "'");
}

const char* to_string(ScheduleStyle style) {
  switch (style) {
    case ScheduleStyle::fsmoe: return "fsmoe";
    case ScheduleStyle::fsmoe_no_iio: return "fsmoe_no_iio";
    case ScheduleStyle::pipemoe: return "pipemoe";
    case ScheduleStyle::sequential: return "sequential";
  }
  return "?";
}

// Kahn sweep over three edge families (explicit deps, per-resource emission
// order, per-order-group emission order). Successor lists keep insertion
// order and the ready set is FIFO, so start times and the busy sums are
// accumulated in the reference's exact order.
Timeline simulate(const Dag& dag) {
  const int n = static_cast<int>(dag.tasks.size());
  std::vector<std::vector<int>> succ(static_cast<size_t>(n));
  std::vector<int> pending(static_cast<size_t>(n), 0);
  auto link = [&](int a, int b) {
    succ[static_cast<size_t>(a)].push_back(b);
    ++pending[static_cast<size_t>(b)];
  };
  std::array<int, 3> lane_tail{-1, -1, -1};
  std::vector<std::pair<int, int>> group_tail;
  for (int i = 0; i < n; ++i) {
    const SimTask& task = dag.tasks[static_cast<size_t>(i)];
    for (int d : task.deps) {
      if (d < 0 || d >= n) throw InvariantError("simulate: dependency on unknown task");
      link(d, i);
    }
    int& tail = lane_tail[static_cast<size_t>(resource_of(task.kind))];
    if (tail >= 0) link(tail, i);
    tail = i;
    if (task.order_group >= 0) {
      auto g = std::find_if(group_tail.begin(), group_tail.end(),
                            [&](const auto& e) { return e.first == task.order_group; });
      if (g == group_tail.end()) {
        group_tail.emplace_back(task.order_group, i);
      } else {
        link(g->second, i);
        g->second = i;
      }
    }
  }
  Timeline tl;
  tl.tasks.assign(static_cast<size_t>(n), ScheduledTask{});
  std::deque<int> fifo;
  for (int i = 0; i < n; ++i)
    if (pending[static_cast<size_t>(i)] == 0) fifo.push_back(i);
  int finished = 0;
  while (!fifo.empty()) {
    const int i = fifo.front();
    fifo.pop_front();
    const SimTask& task = dag.tasks[static_cast<size_t>(i)];
    ScheduledTask& me = tl.tasks[static_cast<size_t>(i)];
    me.end_ms = me.start_ms + task.duration_ms;
    ++finished;
    for (int s : succ[static_cast<size_t>(i)]) {
      ScheduledTask& other = tl.tasks[static_cast<size_t>(s)];
      other.start_ms = std::max(other.start_ms, me.end_ms);
      if (--pending[static_cast<size_t>(s)] == 0) fifo.push_back(s);
    }
    tl.makespan_ms = std::max(tl.makespan_ms, me.end_ms);
    tl.busy_ms[static_cast<size_t>(resource_of(task.kind))] += task.duration_ms;
  }
  if (finished != n) throw InvariantError("simulate: ordering cycle");
  return tl;
}

StageTimes stage_times(const TaskVolumes& vol, const ClusterProfile& profile, int exp_multiplier,
                       int r, std::vector<double> grad_sync_ms) {
  if (r < 1) throw ConfigError("stage_times: degree must be >= 1");
  if (exp_multiplier < 1) throw ConfigError("stage_times: expert multiplier must be >= 1");
  StageTimes st;
  st.degree = r;
  st.dispatch_ms = chunk_ms(profile.a2a, vol.a2a_elements, r);
  st.combine_ms = st.dispatch_ms;
  st.gather_ms = chunk_ms(profile.ag, vol.ag_elements, r);
  st.scatter_ms = chunk_ms(profile.rs, vol.rs_elements, r);
  const LinearModel expert{vol.gemm_count * exp_multiplier * profile.gemm.alpha_ms,
                           vol.gemm_count * exp_multiplier * profile.gemm.beta_ms_per_unit};
  st.expert_ms = chunk_ms(expert, vol.gemm_macs, r);
  st.grad_sync_ms = std::move(grad_sync_ms);
  return st;
}

namespace {

std::string tag(const char* base, int i) { return std::string(base) + "[" + std::to_string(i) + "]"; }

struct DagBuilder {
  Dag& dag;
  int group;  // order group for communication tasks (-1: none)
  int add(OpKind kind, double ms, std::vector<int> deps, std::string label, int chunk, bool comm) {
    SimTask t;
    t.id = static_cast<int>(dag.tasks.size());
    t.kind = kind;
    t.duration_ms = ms;
    t.deps = std::move(deps);
    t.chunk = chunk;
    t.order_group = comm ? group : -1;
    t.label = std::move(label);
    dag.tasks.push_back(t);
    return t.id;
  }
};

struct StageIds {
  std::vector<int> dispatch, gather, expert, scatter, combine, sync;
};

// One pipelined MoE stage: per chunk i dispatch(i) -> gather(i) -> expert(i)
// -> scatter(i) -> combine(i); gradient-sync launches follow the last
// dispatch on the inter link (the post-dispatch slot). `barriers`: each comm
// phase's first task waits for the whole previous phase.
StageIds emit_pipeline(Dag& dag, const StageTimes& s, int group, bool barriers, int base = 0) {
  if (s.degree < 1) throw ConfigError("layer degree must be >= 1");
  DagBuilder b{dag, group};
  StageIds id;
  const int r = s.degree;
  for (int i = 0; i < r; ++i)
    id.dispatch.push_back(b.add(OpKind::a2a_dispatch, s.dispatch_ms, {}, tag("dispatch", i), base + i, true));
  for (size_t j = 0; j < s.grad_sync_ms.size(); ++j)
    id.sync.push_back(b.add(OpKind::grad_allreduce, s.grad_sync_ms[j], {id.dispatch.back()},
                            tag("grad_sync", static_cast<int>(j)), -1, true));
  auto after = [&](const std::vector<int>& prev, int i) {
    if (barriers && i == 0) return prev;
    return std::vector<int>{prev[static_cast<size_t>(i)]};
  };
  for (int i = 0; i < r; ++i)
    id.gather.push_back(b.add(OpKind::allgather, s.gather_ms, after(id.dispatch, i), tag("allgather", i), base + i, true));
  for (int i = 0; i < r; ++i)
    id.expert.push_back(b.add(OpKind::expert, s.expert_ms, {id.gather[static_cast<size_t>(i)]}, tag("expert", i), base + i, false));
  for (int i = 0; i < r; ++i)
    id.scatter.push_back(b.add(OpKind::reducescatter, s.scatter_ms, after(id.expert, i), tag("reducescatter", i), base + i, true));
  for (int i = 0; i < r; ++i)
    id.combine.push_back(b.add(OpKind::a2a_combine, s.combine_ms, after(id.scatter, i), tag("combine", i), base + i, true));
  return id;
}

}  // namespace

Dag build_moe_dag(const StageTimes& stage) {
  Dag dag;
  emit_pipeline(dag, stage, -1, false);
  return dag;
}

Dag build_baseline_dag(ScheduleStyle style, const StageTimes& stage) {
  if (stage.degree < 1) throw ConfigError("layer degree must be >= 1");
  const int r = stage.degree;
  Dag dag;
  switch (style) {
    case ScheduleStyle::fsmoe:
      return build_moe_dag(stage);
    case ScheduleStyle::fsmoe_no_iio:  // one merged comm stream, whole phases
      emit_pipeline(dag, stage, 0, true);
      return dag;
    case ScheduleStyle::pipemoe: {  // interleaved comm, grad sync after all combines
      DagBuilder b{dag, 0};
      std::vector<int> gathers, experts;
      int last_dispatch = -1;
      for (int i = 0; i < r; ++i) {
        last_dispatch = b.add(OpKind::a2a_dispatch, stage.dispatch_ms, {}, tag("dispatch", i), i, true);
        gathers.push_back(b.add(OpKind::allgather, stage.gather_ms, {last_dispatch}, tag("allgather", i), i, true));
      }
      for (int i = 0; i < r; ++i)
        experts.push_back(b.add(OpKind::expert, stage.expert_ms, {gathers[static_cast<size_t>(i)]}, tag("expert", i), i, false));
      for (int i = 0; i < r; ++i) {
        const int rs = b.add(OpKind::reducescatter, stage.scatter_ms, {experts[static_cast<size_t>(i)]}, tag("reducescatter", i), i, true);
        b.add(OpKind::a2a_combine, stage.combine_ms, {rs}, tag("combine", i), i, true);
      }
      for (size_t j = 0; j < stage.grad_sync_ms.size(); ++j)
        b.add(OpKind::grad_allreduce, stage.grad_sync_ms[j], {last_dispatch}, tag("grad_sync", static_cast<int>(j)), -1, true);
      return dag;
    }
    case ScheduleStyle::sequential: {
      DagBuilder b{dag, -1};
      int prev = -1;
      auto chain = [&](OpKind kind, double ms, std::string label, int chunk) {
        std::vector<int> deps;
        if (prev >= 0) deps.push_back(prev);
        prev = b.add(kind, ms, std::move(deps), std::move(label), chunk, false);
      };
      for (int i = 0; i < r; ++i) {
        chain(OpKind::a2a_dispatch, stage.dispatch_ms, tag("dispatch", i), i);
        chain(OpKind::allgather, stage.gather_ms, tag("allgather", i), i);
        chain(OpKind::expert, stage.expert_ms, tag("expert", i), i);
        chain(OpKind::reducescatter, stage.scatter_ms, tag("reducescatter", i), i);
        chain(OpKind::a2a_combine, stage.combine_ms, tag("combine", i), i);
      }
      for (size_t j = 0; j < stage.grad_sync_ms.size(); ++j)
        chain(OpKind::grad_allreduce, stage.grad_sync_ms[j], tag("grad_sync", static_cast<int>(j)), -1);
      return dag;
    }
  }
  throw ConfigError("unknown schedule style");
}

BruteForceResult brute_force_best_degree(const TaskVolumes& vol, const ClusterProfile& profile,
                                         double t_gar_ms, int exp_multiplier, int r_max) {
  if (r_max < 1) throw ConfigError("brute force: r_max must be >= 1");
  BruteForceResult best{1, -1.0};
  for (int r = 1; r <= r_max; ++r) {
    std::vector<double> sync;
    if (t_gar_ms > 0) sync.push_back(t_gar_ms);
    const double ms =
        simulate(build_moe_dag(stage_times(vol, profile, exp_multiplier, r, std::move(sync)))).makespan_ms;
    if (best.makespan_ms < 0 || ms < best.makespan_ms - 1e-15) best = {r, ms};
  }
  return best;
}

double idle_within_span(const Dag& dag, const Timeline& tl, Resource res) {
  double first = -1.0, last = 0.0, busy = 0.0;
  for (size_t i = 0; i < dag.tasks.size(); ++i) {
    if (resource_of(dag.tasks[i].kind) != res) continue;
    if (first < 0 || tl.tasks[i].start_ms < first) first = tl.tasks[i].start_ms;
    last = std::max(last, tl.tasks[i].end_ms);
    busy += dag.tasks[i].duration_ms;
  }
  return first < 0 ? 0.0 : std::max(0.0, (last - first) - busy);
}

namespace {
std::string json_escape(const std::string& s) {
  std::string o;
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o;
}
std::string num(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}
}  // namespace

// Chrome trace-event JSON (schedule_sim.cpp:351-367 fields: name, ph "X",
// ts/dur in microseconds, pid 0, tid = resource lane). The executor's measured
// traces use the same fields so predicted and measured timelines diff.
std::string chrome_trace_json(const Dag& dag, const Timeline& tl) {
  std::string o = "{\n  \"displayTimeUnit\": \"ms\",\n  \"traceEvents\": [";
  for (size_t i = 0; i < dag.tasks.size(); ++i) {
    const SimTask& t = dag.tasks[i];
    o += i ? ",\n    {" : "\n    {";
    o += "\"name\": \"" + json_escape(t.label.empty() ? to_string(t.kind) : t.label) + "\", ";
    o += "\"ph\": \"X\", \"ts\": " + num(tl.tasks[i].start_ms * 1000.0) +
         ", \"dur\": " + num(t.duration_ms * 1000.0) + ", \"pid\": 0, \"tid\": " +
         std::to_string(static_cast<int>(resource_of(t.kind))) + "}";
  }
  o += dag.tasks.empty() ? "]\n}\n" : "\n  ]\n}\n";
  return o;
}

std::string timeline_text(const Dag& dag, const Timeline& tl) {
  std::string out;
  char line[192];
  for (size_t i = 0; i < dag.tasks.size(); ++i) {
    const SimTask& t = dag.tasks[i];
    std::snprintf(line, sizeof line, "%-7s %12.6f %12.6f  %s\n", to_string(resource_of(t.kind)),
                  tl.tasks[i].start_ms, tl.tasks[i].end_ms,
                  t.label.empty() ? to_string(t.kind) : t.label.c_str());
    out += line;
  }
  return out;
}

Dag build_backward_model_dag(const std::vector<BackwardLayerSim>& layers, double tail_sync_ms) {
  Dag dag;
  int prev_combine = -1;
  for (size_t l = 0; l < layers.size(); ++l) {
    const BackwardLayerSim& layer = layers[l];
    std::vector<int> entry;
    if (prev_combine >= 0) entry.push_back(prev_combine);
    DagBuilder b{dag, -1};
    for (size_t j = 0; j < layer.pre_sync_ms.size(); ++j)
      b.add(OpKind::grad_allreduce, layer.pre_sync_ms[j], entry,
            "pre_sync[" + std::to_string(l) + "." + std::to_string(j) + "]", -1, false);
    const int dense = b.add(OpKind::dense_compute, layer.dense_ms, entry,
                            "dense[" + std::to_string(l) + "]", -1, false);
    Dag stage;
    const StageIds ids = emit_pipeline(stage, layer.stage, -1, false, 0);
    const int base = static_cast<int>(dag.tasks.size());
    for (SimTask& t : stage.tasks) {
      t.id += base;
      for (int& d : t.deps) d += base;
      t.label = "L" + std::to_string(l) + "." + t.label;
      dag.tasks.push_back(std::move(t));
    }
    dag.tasks[static_cast<size_t>(base + ids.dispatch.front())].deps.push_back(dense);
    prev_combine = base + ids.combine.back();
  }
  if (tail_sync_ms > 0) {
    DagBuilder b{dag, -1};
    std::vector<int> deps;
    if (prev_combine >= 0) deps.push_back(prev_combine);
    b.add(OpKind::grad_allreduce, tail_sync_ms, deps, "tail_sync", -1, false);
  }
  return dag;
}

// ==================================================== pipeline optimizer ==
// (pipeline_optimizer.cpp:8-213)

LinearModel effective_exp_model(const ClusterProfile& profile, const TaskVolumes& vol,
                                int exp_multiplier) {
  if (vol.gemm_count < 1) throw ConfigError("effective_exp_model: gemm_count must be >= 1");
  if (exp_multiplier < 1) throw ConfigError("effective_exp_model: multiplier must be >= 1");
  return {vol.gemm_count * exp_multiplier * profile.gemm.alpha_ms,
          vol.gemm_count * exp_multiplier * profile.gemm.beta_ms_per_unit};
}

PhaseChunkTimes phase_chunk_times(const PhaseInputs& in, int r) {
  if (r < 1) throw ConfigError("phase_chunk_times: degree must be >= 1");
  PhaseChunkTimes c;
  c.a2a = chunk_ms(in.profile.a2a, in.volumes.a2a_elements, r);
  c.ag = chunk_ms(in.profile.ag, in.volumes.ag_elements, r);
  c.rs = chunk_ms(in.profile.rs, in.volumes.rs_elements, r);
  c.exp = chunk_ms(effective_exp_model(in.profile, in.volumes, in.exp_multiplier),
                   in.volumes.gemm_macs, r);
  return c;
}

// Q1..Q7 (§4): strict inequalities between chunk times and the
// gradient-sync budget G; evaluated exactly as the reference writes them.
PredicateVector q_predicates(const PhaseInputs& in, int r) {
  const PhaseChunkTimes c = phase_chunk_times(in, r);
  const double G = in.t_gar_ms;
  const double overlap = 2 * (r - 1) * c.a2a;  // return-stream exposure of r-1 chunks
  PredicateVector q;
  q[0] = c.a2a > c.ag;
  q[1] = r * c.exp > overlap;
  q[2] = r * c.exp > (r - 1) * (c.ag + c.rs);
  q[3] = G > c.ag + c.rs;
  q[4] = G > r * c.exp - overlap + c.ag + c.rs;
  q[5] = G > r * c.ag + r * c.rs - overlap;
  q[6] = G > c.ag + c.rs + r * c.exp - overlap;
  return q;
}

bool case_feasible(int case_id, const PredicateVector& q) {
  const bool a = q[0], b = q[1], c = q[2], d = q[3], e = q[4], f = q[5], g = q[6];
  if (case_id == 1) return (a && !b && d) || (a && b && e) || (!a && !c && f) || (!a && c && g);
  if (case_id == 2) return (a && b && !e) || (!a && c && !g);
  if (case_id == 3) return a && !b && !d;
  if (case_id == 4) return !a && !c && !f;
  throw InvariantError("case_feasible: unknown case id");
}

double case_cost(int case_id, const PhaseInputs& in, int r) {
  const PhaseChunkTimes c = phase_chunk_times(in, r);
  if (case_id == 1) return 2 * r * c.a2a + in.t_gar_ms;       // inter-link bound, sync exposed
  if (case_id == 2) return 2 * c.a2a + c.ag + c.rs + r * c.exp;  // expert bound
  if (case_id == 3) return 2 * r * c.a2a + c.ag + c.rs;        // AlltoAll bound
  if (case_id == 4) return 2 * c.a2a + r * (c.ag + c.rs);      // intra-collective bound
  throw InvariantError("case_cost: unknown case id");
}

CaseMin minimize_case(int case_id, const PhaseInputs& in, int r_max) {
  if (r_max < 1) throw ConfigError("minimize_case: r_max must be >= 1");
  CaseMin best;
  for (int r = 1; r <= r_max; ++r) {
    if (!case_feasible(case_id, q_predicates(in, r))) continue;
    const double t = case_cost(case_id, in, r);
    if (!best.feasible || t < best.t_ms) best = {true, r, t};
  }
  return best;
}

DegreeChoice find_optimal_pipeline_degree(const PhaseInputs& in, int r_max) {
  DegreeChoice ch;
  bool found = false;
  for (int k = 1; k <= 4; ++k) {
    const CaseMin m = minimize_case(k, in, r_max);
    if (!m.feasible) continue;
    const bool wins = !found || m.t_ms < ch.t_moe_ms ||
                      (m.t_ms == ch.t_moe_ms && (m.r < ch.r || (m.r == ch.r && k < ch.case_id)));
    if (wins) {
      ch.r = m.r;
      ch.case_id = k;
      ch.t_moe_ms = m.t_ms;
      found = true;
    }
  }
  const LinearModel& ag = in.profile.ag;
  const LinearModel& rs = in.profile.rs;
  if (!found) {
    // unreachable while the regions partition the predicate space
    const BruteForceResult bf =
        brute_force_best_degree(in.volumes, in.profile, in.t_gar_ms, in.exp_multiplier, r_max);
    ch.r = bf.r;
    ch.case_id = 0;
    ch.t_moe_ms = bf.makespan_ms;
    ch.boundary = true;
  } else if (ag.alpha_ms != rs.alpha_ms || ag.beta_ms_per_unit != rs.beta_ms_per_unit) {
    // asymmetric collectives: polish the analytic degree with simulation
    std::vector<double> sync;
    if (in.t_gar_ms > 0) sync.push_back(in.t_gar_ms);
    auto simulated = [&](int r) {
      return simulate(build_moe_dag(stage_times(in.volumes, in.profile, in.exp_multiplier, r, sync)))
          .makespan_ms;
    };
    double best_ms = simulated(ch.r);
    int best_r = ch.r;
    for (int r = 1; r <= r_max; ++r) {
      if (r == ch.r) continue;
      const double ms = simulated(r);
      if (ms < best_ms * (1.0 - 1e-9)) {
        best_ms = ms;
        best_r = r;
      }
    }
    if (best_r != ch.r) {
      const PredicateVector qr = q_predicates(in, best_r);
      ch.r = best_r;
      ch.case_id = 0;
      for (int k = 1; k <= 4 && ch.case_id == 0; ++k)
        if (case_feasible(k, qr)) ch.case_id = k;
      ch.t_moe_ms = ch.case_id ? case_cost(ch.case_id, in, best_r) : best_ms;
      ch.boundary = ch.case_id == 0;
    }
  }
  ch.q = q_predicates(in, ch.r);
  return ch;
}

double overlappable_moe_time(int case_id, const PhaseInputs& in, int r) {
  const PhaseChunkTimes c = phase_chunk_times(in, r);
  if (case_id == 2) return std::max(0.0, r * c.exp + c.ag + c.rs - 2 * (r - 1) * c.a2a);
  if (case_id == 3) return std::max(0.0, c.ag + c.rs);
  if (case_id == 4) return std::max(0.0, r * (c.ag + c.rs) - 2 * (r - 1) * c.a2a);
  throw InvariantError(
      "overlappable_moe_time: only the compute- and collective-bound cases expose inter-link "
      "idle");
}

PipelinePlan plan_layer(const TaskVolumes& vol, const ClusterProfile& profile, double t_gar_bwd_ms,
                        int r_max) {
  PhaseInputs fwd{vol, profile, 0.0, 1};
  PhaseInputs bwd{vol, profile, t_gar_bwd_ms, 2};
  PipelinePlan p;
  const DegreeChoice f = find_optimal_pipeline_degree(fwd, r_max);
  p.r_fwd = f.r;
  p.case_fwd = f.case_id;
  p.t_moe_fwd_ms = f.t_moe_ms;
  p.q_fwd = f.q;
  p.boundary_fwd = f.boundary;
  const DegreeChoice b = find_optimal_pipeline_degree(bwd, r_max);
  p.r_bwd = b.r;
  p.case_bwd = b.case_id;
  p.t_moe_bwd_ms = b.t_moe_ms;
  p.q_bwd = b.q;
  p.boundary_bwd = b.boundary;
  p.t_gar_bwd_ms = t_gar_bwd_ms;
  // inter-link idle at the chosen backward degree with the sync removed; the
  // last feasible case wins, as in the reference
  PhaseInputs open = bwd;
  open.t_gar_ms = 0.0;
  const PredicateVector q0 = q_predicates(open, p.r_bwd);
  int last = 0;
  for (int k = 1; k <= 4; ++k)
    if (case_feasible(k, q0)) last = k;
  p.t_olp_moe_bwd_ms = last >= 2 ? overlappable_moe_time(last, open, p.r_bwd) : 0.0;
  return p;
}

// ================================================== gradient partitioning ==
// (grad_partition.cpp:11-228)

namespace {

bool moves_tokens(const TaskVolumes& v) {
  return v.a2a_elements > 0 || v.ag_elements > 0 || v.rs_elements > 0 || v.gemm_macs > 0;
}

// Backward span of a layer carrying a sync launch of t_gar; a layer without
// expert traffic exposes the launch bare.
double span_with_sync(const GradLayer& layer, const ClusterProfile& profile, double t_gar,
                      int r_max) {
  if (!moves_tokens(layer.volumes)) return t_gar;
  return find_optimal_pipeline_degree(PhaseInputs{layer.volumes, profile, t_gar, 2}, r_max).t_moe_ms;
}

double allreduce_ms(const ClusterProfile& profile, double elements) {
  return elements > 0 ? predict_ms(profile.ar, elements) : 0.0;
}

// Project x onto the availability polytope: slot i carries at most the
// gradient produced up to layer i and not yet assigned.
void clamp_to_available(std::vector<double>& x, const std::vector<double>& remainder) {
  double avail = 0.0;
  for (size_t i = 0; i < x.size(); ++i) {
    avail += remainder[i];
    x[i] = std::clamp(x[i], 0.0, avail);
    avail -= x[i];
  }
}

}  // namespace

SyncWindow sync_window(const GradLayer& layer, const ClusterProfile& profile, int r_max) {
  SyncWindow w;
  w.t_olp_dense_ms = layer.t_olp_dense_ms;
  if (!moves_tokens(layer.volumes)) return w;
  const PhaseInputs in{layer.volumes, profile, 0.0, 2};
  const DegreeChoice d = find_optimal_pipeline_degree(in, r_max);
  w.degree = d.r;
  w.case_id = d.case_id;
  w.t_olp_moe_ms = d.case_id >= 2 ? overlappable_moe_time(d.case_id, in, d.r) : 0.0;
  return w;
}

Step1Result step1_assign(const std::vector<GradLayer>& layers, const ClusterProfile& profile,
                         const std::vector<SyncWindow>& windows) {
  if (windows.size() != layers.size()) throw ConfigError("step1: one window per layer required");
  const size_t n = layers.size();
  Step1Result r;
  r.n_first.assign(n, 0.0);
  r.n_first_dense.assign(n, 0.0);
  r.n_first_moe.assign(n, 0.0);
  std::vector<double> waiting(n, 0.0);  // produced, not yet absorbed, by origin layer
  for (size_t i = 0; i < n; ++i) {
    double room_dense = invert_elements(profile.ar, windows[i].t_olp_dense_ms);
    double room_moe = invert_elements(profile.ar, windows[i].t_olp_moe_ms);
    for (size_t j = 0; j < i; ++j) {  // oldest origin first
      if (waiting[j] <= 0) continue;
      const double a = std::min(room_dense, waiting[j]);
      room_dense -= a;
      waiting[j] -= a;
      r.n_first_dense[i] += a;
      const double b = std::min(room_moe, waiting[j]);
      room_moe -= b;
      waiting[j] -= b;
      r.n_first_moe[i] += b;
      if (room_dense <= 0 && room_moe <= 0) break;
    }
    r.n_first[i] = r.n_first_dense[i] + r.n_first_moe[i];
    waiting[i] = layers[i].n_grad;  // this layer's own gradient joins afterwards
  }
  r.remainder = waiting;
  return r;
}

// Differential evolution rand/1/bin with repair (§5 step 2).
std::vector<double> step2_optimize(const std::vector<GradLayer>& layers,
                                   const std::vector<double>& remainder,
                                   const ClusterProfile& profile, const DeParams& de, int r_max,
                                   const std::vector<double>& slot_base) {
  const size_t dims = layers.size();
  if (remainder.size() != dims) throw ConfigError("step2: one remainder entry per layer required");
  if (!slot_base.empty() && slot_base.size() != dims)
    throw ConfigError("step2: one slot base entry per layer required");
  if (dims == 0) return {};
  double total_rem = 0.0;
  for (double v : remainder) total_rem += v;
  auto cost = [&](const std::vector<double>& x) {
    double spans = 0.0, placed = 0.0;
    for (size_t i = 0; i < dims; ++i) {
      const double base = slot_base.empty() ? 0.0 : slot_base[i];
      spans += span_with_sync(layers[i], profile, allreduce_ms(profile, base + x[i]), r_max);
      placed += x[i];
    }
    return spans + allreduce_ms(profile, total_rem - placed);
  };
  const int np = de.population > 0 ? de.population : std::max<int>(8, 15 * static_cast<int>(dims));
  if (np < 4) throw ConfigError("step2: population must be at least 4");
  if (de.generations < 0) throw ConfigError("step2: negative generations");
  std::mt19937_64 gen(de.seed);
  auto u01 = [&] { return (gen() >> 11) * 0x1.0p-53; };
  std::vector<std::vector<double>> pop(static_cast<size_t>(np), std::vector<double>(dims, 0.0));
  pop[1] = remainder;  // member 0: all to the tail; member 1: every remainder in its slot
  for (size_t m = 2; m < pop.size(); ++m)
    for (size_t i = 0; i < dims; ++i) pop[m][i] = u01() * remainder[i];
  for (auto& member : pop) clamp_to_available(member, remainder);
  std::vector<double> fit(pop.size());
  for (size_t m = 0; m < pop.size(); ++m) fit[m] = cost(pop[m]);
  std::vector<double> cand(dims);
  const size_t P = pop.size();
  for (int g = 0; g < de.generations; ++g) {
    for (size_t m = 0; m < P; ++m) {
      size_t a, b, c;
      do a = gen() % P; while (a == m);
      do b = gen() % P; while (b == m || b == a);
      do c = gen() % P; while (c == m || c == a || c == b);
      const size_t forced = gen() % dims;
      for (size_t i = 0; i < dims; ++i) {
        const bool mutate = u01() < de.crossover || i == forced;
        cand[i] = mutate ? pop[a][i] + de.weight * (pop[b][i] - pop[c][i]) : pop[m][i];
      }
      clamp_to_available(cand, remainder);
      const double f = cost(cand);
      if (f <= fit[m]) {
        pop[m] = cand;
        fit[m] = f;
      }
    }
  }
  size_t best = 0;
  for (size_t m = 1; m < P; ++m)
    if (fit[m] < fit[best]) best = m;
  return pop[best];
}

PartitionPlan build_partition_plan(const std::vector<GradLayer>& layers,
                                   const ClusterProfile& profile, const DeParams& de, int r_max) {
  const size_t n = layers.size();
  std::vector<SyncWindow> windows;
  windows.reserve(n);
  for (const GradLayer& l : layers) windows.push_back(sync_window(l, profile, r_max));
  const Step1Result s1 = step1_assign(layers, profile, windows);
  double rem = 0.0;
  for (double v : s1.remainder) rem += v;
  PartitionPlan plan;
  std::vector<double> x(n, 0.0);
  if (rem > 0) {
    x = step2_optimize(layers, s1.remainder, profile, de, r_max, s1.n_first_moe);
    plan.step2_ran = true;
  }
  double tail = 0.0, objective = 0.0;
  plan.layers.resize(n);
  for (size_t i = 0; i < n; ++i) {
    LayerAssignment& a = plan.layers[i];
    a.n_first = s1.n_first[i];
    a.n_first_dense = s1.n_first_dense[i];
    a.n_first_moe = s1.n_first_moe[i];
    a.x_g = x[i];
    a.window = windows[i];
    const double load = a.n_first + a.x_g;
    a.t_gar_ms = load > 0 ? predict_ms(profile.ar, load) : 0.0;
    tail += s1.remainder[i];  // replaying the repair recurrence keeps tail >= 0 exactly
    tail -= x[i];
    objective += span_with_sync(layers[i], profile, allreduce_ms(profile, s1.n_first_moe[i] + x[i]), r_max);
  }
  plan.tail_elements = tail;
  plan.tail_ms = allreduce_ms(profile, plan.tail_elements);
  plan.objective_ms = objective + plan.tail_ms;
  return plan;
}

}  // namespace fsmoe
