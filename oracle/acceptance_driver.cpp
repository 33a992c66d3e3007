// ORACLE / test infrastructure only.
//
// Runs selected criteria of the reference's acceptance program
// (/root/reference/proj/tests/acceptance.cpp, included UNMODIFIED below, its own
// main() renamed away) so a test can pick the criteria that exercise the
// Net / Solver hot path without the ones that need the reference CLI
// (8: CLI determinism, 9: CLI bench row), which is not built here.
//
//   acceptance_{ref,b200} [criterion numbers 1..9 ...]   (default: 1 2 3 5 6 7)
// Prints "PASS i/9 name: detail" / "FAIL ..." per criterion, exits with the
// number of failures.
#define main reference_acceptance_main
#include "acceptance.cpp"
#undef main

#include <cstdlib>

int main(int argc, char** argv) {
  const struct {
    const char* name;
    Outcome (*run)();
  } criteria[] = {
      {"scalar policy head worked-example arithmetic", check_sigmoid_head_arithmetic},
      {"distribution policy head worked-example arithmetic", check_softmax_head_arithmetic},
      {"finite-difference gradient checks", check_gradients},
      {"cart-pole policies learn to balance", check_cartpole_learning},
      {"model files round-trip through the parser", check_prototxt_round_trip},
      {"sampler statistics match their design", check_sampler_statistics},
      {"cart-pole dynamics match hand-computed values", check_dynamics},
      {"training CLI is deterministic per seed", check_cli_determinism},
      {"benchmark output and dispatch equivalence", check_bench_and_dispatch},
  };
  std::vector<int> pick;
  for (int i = 1; i < argc; ++i) pick.push_back(std::atoi(argv[i]));
  if (pick.empty()) pick = {1, 2, 3, 5, 6, 7};
  int failures = 0;
  for (int idx : pick) {
    if (idx < 1 || idx > 9) {
      std::printf("FAIL %d/9 no such criterion\n", idx);
      ++failures;
      continue;
    }
    Outcome outcome;
    try {
      outcome = criteria[idx - 1].run();
    } catch (const std::exception& e) {
      outcome = {false, std::string("exception: ") + e.what()};
    }
    if (!outcome.pass) ++failures;
    std::printf("%s %d/9 %s: %s\n", outcome.pass ? "PASS" : "FAIL", idx, criteria[idx - 1].name,
                outcome.detail.c_str());
    std::fflush(stdout);
  }
  return failures;
}
