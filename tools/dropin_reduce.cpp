// Drop-in demonstration: the reference CLI's `reduce` command
// (/root/reference/proj/tools/main.cpp:52-120, cmd_reduce) written against
// include/kronred_b200.hpp instead of the reference headers. The calls, types
// and outputs are the reference's; only the include and the link line change:
//
//   g++ -std=c++20 -O2 -Iinclude tools/dropin_reduce.cpp \
//       -Lpaper_2510_19608_b200/_lib -lkronred_b200 \
//       -Wl,-rpath,$PWD/paper_2510_19608_b200/_lib -o dropin_reduce
//
//   ./dropin_reduce net.json scen.csv e_bar [mag|complex] [target] [--radialize]
//                   [reduced.json] [trace.csv]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <optional>
#include <string>

#include "kronred_b200.hpp"

using namespace kronred;

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s net.json scen.csv e_bar [mag|complex] [target|-] [--radialize] [out.json] [trace.csv]\n",
                 argv[0]);
    return 2;
  }
  try {
    const Network net = read_network_json(argv[1]);
    validate_or_throw(net);
    const ScenarioLibrary lib = load_library(net, argv[2]);

    ReductionConfig cfg;
    cfg.e_bar = std::strtod(argv[3], nullptr);
    const std::string obj = argc > 4 ? argv[4] : "mag";
    if (obj == "mag")
      cfg.objective = Objective::magnitude;
    else if (obj == "complex")
      cfg.objective = Objective::complex_error;
    else
      throw ConfigError("--objective must be 'mag' or 'complex'");
    if (argc > 5 && std::strcmp(argv[5], "-") != 0) cfg.target_reduction = std::strtod(argv[5], nullptr);
    const bool radial = argc > 6 && std::strcmp(argv[6], "--radialize") == 0;
    const std::string out_reduced = argc > 7 ? argv[7] : "reduced.json";
    const std::string out_trace = argc > 8 ? argv[8] : "trace.csv";

    ReductionResult result = run_reduction(net, lib, cfg);
    ReducedModel model = std::move(result.model);
    if (radial) {
      const BlockAdmittance y = assemble_admittance(net);
      model = radialize(model, net, y, &lib);
    }
    write_reduced_json(model, out_reduced);
    write_trace_csv(out_trace, result.trace, model.scenario_ids, model.final_max_err);

    const int n = net.size();
    const int kept = int(model.kept_ids.size());
    std::printf("reduced %d -> %d nodes (%.1f%% reduction, %zu iterations)\n", n, kept,
                100.0 * double(n - kept) / double(n), result.trace.size());
    for (size_t l = 0; l < model.final_max_err.size(); ++l)
      std::cout << "  max |dV| " << model.scenario_ids[l] << ": " << format_double(model.final_max_err[l]) << "\n";
    return 0;
  } catch (const SolverError& e) {
    std::cerr << "SolverError: " << e.what() << "\n";
    return 3;
  } catch (const Error& e) {
    std::cerr << e.what() << "\n";
    return 2;
  }
}
