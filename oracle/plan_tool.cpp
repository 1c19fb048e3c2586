// oracle/plan_tool.cpp — TEST-ONLY golden generator for the planner
// interchange formats (paper_2501_10714_b200/planio.py). Links the
// reference's own planner + json_io sources, compiled in place from
// /root/reference/proj/src (never copied), and prints the documents the
// reference CLI's fit / plan / simulate subcommands would write
// (cli/main.cpp:79-210; that CLI itself needs CLI11, absent here, so this
// driver stands in for its argument parsing). Output -> tests/golden/planio/.
//
//   plan_tool fit <bench.csv> <min_r2>
//   plan_tool plan <model.json> <profile.json>
//   plan_tool simulate <model.json> <profile.json> <style> <fwd|bwd> <layer>
#include <cstdio>
#include <iostream>
#include <string>
#include <vector>

#include "fsmoe/cost_models.hpp"
#include "fsmoe/grad_partition.hpp"
#include "fsmoe/json_io.hpp"
#include "fsmoe/pipeline_optimizer.hpp"
#include "fsmoe/schedule_sim.hpp"
#include "fsmoe/workload.hpp"

using fsmoe::json;

static json vol_doc(const fsmoe::TaskVolumes& v) {
  return json{{"a2a_elements", v.a2a_elements}, {"ag_elements", v.ag_elements},
              {"rs_elements", v.rs_elements},   {"gemm_macs", v.gemm_macs},
              {"gemm_count", v.gemm_count},     {"grad_elements", v.grad_elements},
              {"capacity", v.capacity}};
}

int main(int argc, char** argv) {
  try {
    const std::string mode = argc > 1 ? argv[1] : "";
    if (mode == "fit" && argc == 4) {
      auto fit = fsmoe::fit_profile(fsmoe::load_bench_csv(argv[2]), std::stod(argv[3]));
      json doc = fsmoe::profile_to_json(fit.profile);
      doc["fit"] = json{{"min_r_squared", fit.min_r_squared}, {"clamped_kinds", fit.clamped_kinds}};
      std::cout << doc.dump(2) << "\n";
      return 0;
    }
    if (mode == "plan" && argc == 4) {
      auto model = fsmoe::load_model(argv[2]);
      auto prof = fsmoe::load_profile(argv[3]);
      std::vector<fsmoe::TaskVolumes> vols;
      std::vector<fsmoe::GradLayer> grads;
      for (const auto& l : model.layers) {
        vols.push_back(fsmoe::derive_volumes(l, model.parallel));
        grads.push_back(fsmoe::GradLayer{vols.back(), l.t_olp_dense_ms, vols.back().grad_elements});
      }
      auto part = fsmoe::build_partition_plan(grads, prof, model.de, model.r_max);
      json doc;
      doc["r_max"] = model.r_max;
      doc["seed"] = model.de.seed;
      doc["layers"] = json::array();
      for (size_t i = 0; i < vols.size(); ++i) {
        auto p = fsmoe::plan_layer(vols[i], prof, part.layers[i].t_gar_ms, model.r_max);
        doc["layers"].push_back(json{{"index", static_cast<int>(i)}, {"volumes", vol_doc(vols[i])},
                                     {"pipeline", fsmoe::plan_to_json(p)}});
      }
      doc["partition"] = fsmoe::partition_to_json(part);
      std::cout << doc.dump(2) << "\n";
      return 0;
    }
    if (mode == "simulate" && argc == 7) {
      auto model = fsmoe::load_model(argv[2]);
      auto prof = fsmoe::load_profile(argv[3]);
      auto style = fsmoe::style_from_string(argv[4]);
      const std::string pass = argv[5];
      const int li = std::stoi(argv[6]);
      auto vol = fsmoe::derive_volumes(model.layers.at(li), model.parallel);
      double t_gar = (pass == "bwd" && vol.grad_elements > 0) ? fsmoe::predict_ms(prof.ar, vol.grad_elements) : 0.0;
      auto plan = fsmoe::plan_layer(vol, prof, t_gar, model.r_max);
      const int r = pass == "fwd" ? plan.r_fwd : plan.r_bwd;
      std::vector<double> sync;
      if (t_gar > 0) sync.push_back(t_gar);
      auto tl = fsmoe::simulate(fsmoe::build_baseline_dag(
          style, fsmoe::stage_times(vol, prof, pass == "fwd" ? 1 : 2, r, sync)));
      json doc{{"style", fsmoe::to_string(style)}, {"pass", pass}, {"layer", li}, {"r", r},
               {"makespan_ms", tl.makespan_ms}};
      json busy, util;
      for (auto res : {fsmoe::Resource::inter_link, fsmoe::Resource::intra_link, fsmoe::Resource::compute}) {
        const double b = tl.busy_ms[static_cast<int>(res)];
        busy[fsmoe::to_string(res)] = b;
        util[fsmoe::to_string(res)] = tl.makespan_ms > 0 ? b / tl.makespan_ms : 0.0;
      }
      doc["busy_ms"] = busy;
      doc["utilization"] = util;
      std::cout << doc.dump(2) << "\n";
      return 0;
    }
    std::fprintf(stderr, "usage: plan_tool fit|plan|simulate ...\n");
    return 2;
  } catch (const fsmoe::ConfigError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const fsmoe::FitQualityError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  }
}
