// The reference's verification suite (src/verify/verify.cpp, run_verify_suite
// :345-399 -- what `jigsaw verify` runs) as a standalone program, linked
// against the B200 drop-in (jigsaw_spb_b200.cpp) instead of the reference's
// src/spb/{spb,model}.cpp. The reference's CLI (CLI11, not vendored) is not
// needed: this is its verify sub-command's loop (jigsaw_main.cpp:136-145).
//   verify_gpu [k B trials sgd_iterations seed]
#include <cstdio>
#include <cstdlib>

#include "jigsaw/verify/verify.hpp"

int main(int argc, char** argv) {
  jigsaw::verify::VerifyOptions opts;
  if (argc > 1) opts.k = std::atoi(argv[1]);
  if (argc > 2) opts.B = std::atoi(argv[2]);
  if (argc > 3) opts.trials = std::atoi(argv[3]);
  if (argc > 4) opts.sgd_iterations = std::atoi(argv[4]);
  if (argc > 5) opts.seed = std::strtoull(argv[5], nullptr, 10);
  int failed = 0, total = 0;
  for (const auto& r : jigsaw::verify::run_verify_suite(opts)) {
    std::printf("[%s] %s %s\n", r.pass ? "PASS" : "FAIL", r.name.c_str(), r.detail.c_str());
    ++total;
    if (!r.pass) ++failed;
  }
  std::printf("verify: %d/%d checks passed\n", total - failed, total);
  return failed ? 1 : 0;
}
