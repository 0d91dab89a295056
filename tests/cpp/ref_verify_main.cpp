// tests/cpp/ref_verify_main.cpp -- drives the reference's OWN acceptance suite
// (proj/src/runner.cpp run_verify + check_accuracy_sanity +
// check_baseline_kernel_divergence, compiled unmodified from /root/reference by
// tests/cpp/Makefile) against the drop-in headers include/tbik/{errors,numerics,
// rng,matrix,matmul,collective,layers}.hpp and libtbik_b200: every
// tree_matmul / row_parallel_forward / column_parallel_forward / tree_all_reduce
// / baseline_* call the reference's checks make runs on the B200.  The
// reference's non-hot-path files (oracle.cpp, witness.cpp, report.cpp,
// threading.cpp, demo.cpp) are linked as they are, as the callers.
#include <cstdio>

#include "tbik/runner.hpp"

int main() {
  try {
    tbik::VerifyOptions opts;  // the reference defaults: tp 1/2/4/8, batch 8/16/32, 5 seeds, 64x4096x128
    opts.dtypes = {tbik::Dtype::Bf16, tbik::Dtype::F32};
    tbik::RunReport report = tbik::run_verify(opts);
    report.add(tbik::check_accuracy_sanity(3));
    report.add(tbik::check_baseline_kernel_divergence(1, opts.tp_set));
    report.add(tbik::check_bf16_exhaustive());
    std::printf("%s", report.to_string(true).c_str());
    for (const auto& c : report.checks)
      std::printf("%s %s %s\n", c.pass ? "PASS" : "FAIL", c.name.c_str(), c.detail.c_str());
    std::printf("%s\n", report.all_passed() ? "ALL PASS" : "SOME FAILED");
    return report.all_passed() ? 0 : 1;
  } catch (const tbik::TbikError& e) {
    std::printf("FAIL exception %s (status %d)\n", e.what(), e.status());
    return 2;
  }
}
