// SPDX-License-Identifier: Apache-2.0
//
// seqbal -- command-line front end, the reference CLI's `plan` subcommand
// (proj/tools/main.cpp:200-230, options :344-351, exit codes :369-387):
//
//   seqbal plan LENS_FILE --topology SPEC [--d-model 3072] [--n-heads 24] [--gamma 0.49]
//
// reads a JSON array of per-rank length arrays, plans on the GPU through the
// C++ drop-in API (plan_routing in libseqbal.so -> libseqbal_cuda.so) and
// prints plan_to_json, byte-identical to the reference CLI.  Errors: "error:
// ..." and exit 1 (ConfigError / ParseError / bad arguments); "invariant
// violation: ..." and exit 2 (IntegrityError).
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "seqbal/seqbal.hpp"

namespace seqbal {
std::vector<std::vector<std::int64_t>> read_lens_json(const std::string& text);
}

namespace {

int usage(const char* why) {
  std::cerr << "error: " << why << "\n"
            << "usage: seqbal plan LENS_FILE --topology SPEC [--d-model N] [--n-heads N] [--gamma G]\n";
  return 1;
}

int cmd_plan(const std::string& lens_file, const std::string& topo, int d_model, int n_heads, double gamma) {
  using namespace seqbal;
  std::ifstream in(lens_file);
  if (!in) throw ConfigError("cannot open seq-lens file: " + lens_file);
  std::stringstream ss;
  ss << in.rdbuf();
  const auto lens = read_lens_json(ss.str());
  std::vector<std::vector<SequenceInfo>> per_rank;
  std::uint64_t id = 0;
  for (const auto& r : lens) {
    std::vector<SequenceInfo> seqs;
    for (std::int64_t l : r) seqs.push_back({id++, l});
    per_rank.push_back(std::move(seqs));
  }
  WorkloadModel model;
  if (n_heads <= 0 || d_model % n_heads != 0) throw ConfigError("d_model must be divisible by n_heads");
  model.shape = ModelShape{d_model, n_heads, d_model / n_heads, 1};
  model.gamma = gamma;
  const Topology topology = parse_topology(topo);
  const WorldLayout layout = replicate(topology, static_cast<int>(per_rank.size()));
  const PlanResult result = plan_routing(per_rank, model, layout);
  std::cout << plan_to_json(result.plan, result.report) << "\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage("a subcommand is required (plan)");
  const std::string sub = argv[1];
  if (sub != "plan") return usage(("unknown subcommand '" + sub + "'").c_str());
  std::string file, topo;
  int d_model = 3072, n_heads = 24;
  double gamma = seqbal::kGammaH100;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&](const char* name) -> std::string {
      if (i + 1 >= argc) throw std::invalid_argument(std::string(name) + " requires a value");
      return argv[++i];
    };
    try {
      if (a == "--topology") topo = val("--topology");
      else if (a == "--d-model") d_model = std::stoi(val("--d-model"));
      else if (a == "--n-heads") n_heads = std::stoi(val("--n-heads"));
      else if (a == "--gamma") gamma = std::stod(val("--gamma"));
      else if (!a.empty() && a[0] == '-') return usage(("unknown option " + a).c_str());
      else if (file.empty()) file = a;
      else return usage("too many positional arguments");
    } catch (const std::exception& e) {
      return usage(e.what());
    }
  }
  if (file.empty()) return usage("lens-file is required");
  if (topo.empty()) return usage("--topology is required");
  try {
    return cmd_plan(file, topo, d_model, n_heads, gamma);
  } catch (const seqbal::IntegrityError& e) {
    std::cerr << "invariant violation: " << e.what() << "\n";
    return 2;
  } catch (const std::invalid_argument& e) {  // ConfigError, ParseError
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
