// qsim — scenario runner CLI (the reference's tools/qsim.cpp:34-102): `qsim run <spec>
// [--out-dir D] [--seed S] [--ntraj N] [--threads T]`, `qsim list`, `qsim validate <spec>`.
// Same subcommands, options, outputs and exit codes (0 ok, 2 invalid spec, 3 solver failure);
// the solves run on the GPU through the qsim C++ API. CLI11 (a vendored header the reference
// uses) is not shipped, so the arguments are parsed by hand.
#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <iostream>
#include <optional>
#include <string>
#include <vector>

#include "../../../include/qsim/qobj.hpp"
#include "../../../include/qsim/scenario.hpp"

namespace {

// an existing file path wins, otherwise a built-in name with or without ".json" (tools/qsim.cpp:12-22)
qsim::ScenarioSpec resolve_scenario(const std::string& arg) {
  if (std::filesystem::exists(arg)) return qsim::load_scenario_file(arg);
  std::string name = arg;
  if (name.size() > 5 && name.ends_with(".json")) name = name.substr(0, name.size() - 5);
  if (const std::string* text = qsim::builtin_scenario_json(name)) return qsim::parse_scenario(*text);
  qsim::throw_error(qsim::ErrorCode::InvalidScenario, "no such scenario file or built-in: " + arg);
}

int default_threads() {  // tools/qsim.cpp:24-30
  if (const char* env = std::getenv("QSIM_THREADS")) {
    const int n = std::atoi(env);
    if (n > 0) return n;
  }
  return 0;
}

int usage(int rc) {
  std::cerr << "qsim - open quantum system scenario runner (B200)\n"
               "usage: qsim run <spec> [--out-dir DIR] [--seed S] [--ntraj N] [--threads T]\n"
               "       qsim list\n"
               "       qsim validate <spec>\n";
  return rc;
}

}  // namespace

int main(int argc, char** argv) {
  std::vector<std::string> args(argv + 1, argv + argc);
  if (args.empty()) return usage(109);  // CLI11's RequiredError exit code for a missing subcommand
  const std::string cmd = args[0];
  try {
    if (cmd == "list") {
      for (const auto& name : qsim::builtin_scenario_names()) std::cout << name << "\n";
      return 0;
    }
    if (cmd == "validate") {
      if (args.size() < 2) return usage(109);
      qsim::ScenarioSpec spec = resolve_scenario(args[1]);
      auto diags = qsim::validate(spec);
      if (diags.empty()) {
        std::cout << "{\"valid\":true,\"diagnostics\":[]}\n";
        return 0;
      }
      std::cout << "{\"valid\":false,\"diagnostics\":[";
      for (size_t i = 0; i < diags.size(); ++i) std::cout << '"' << diags[i] << (i + 1 < diags.size() ? "\"," : "\"");
      std::cout << "]}\n";
      return 2;
    }
    if (cmd != "run") return usage(109);
    std::string spec_arg;
    qsim::RunOverrides overrides;
    std::optional<int> threads;
    for (size_t i = 1; i < args.size(); ++i) {
      const std::string& a = args[i];
      auto value = [&]() -> std::string {
        if (i + 1 >= args.size()) throw std::invalid_argument(a + " needs a value");
        return args[++i];
      };
      if (a == "--out-dir") overrides.out_dir = value();
      else if (a == "--seed") overrides.seed = std::stoull(value());
      else if (a == "--ntraj") overrides.ntraj = std::stoi(value());
      else if (a == "--threads") threads = std::stoi(value());
      else if (!a.empty() && a[0] == '-') throw std::invalid_argument("unknown option " + a);
      else spec_arg = a;
    }
    if (spec_arg.empty()) return usage(109);
    if (threads) overrides.n_threads = *threads;
    else if (int n = default_threads(); n > 0) overrides.n_threads = n;
    qsim::ScenarioSpec spec = resolve_scenario(spec_arg);
    qsim::RunOutcome outcome = qsim::run_scenario(spec, overrides);
    if (outcome.exit_code != 0) {
      std::cerr << outcome.error_json << "\n";
      return outcome.exit_code;
    }
    std::cout << "wrote " << outcome.csv_path << " and " << outcome.json_path << "\n";
    return 0;
  } catch (const qsim::Error& e) {
    std::cerr << "{\"error\":\"" << qsim::error_code_name(e.code()) << "\",\"message\":\"" << e.what() << "\"}\n";
    return e.code() == qsim::ErrorCode::InvalidScenario ? 2 : 3;
  } catch (const std::invalid_argument& e) {
    std::cerr << e.what() << "\n";
    return usage(109);
  } catch (const std::exception& e) {
    std::cerr << "{\"error\":\"exception\",\"message\":\"" << e.what() << "\"}\n";
    return 3;
  }
}
