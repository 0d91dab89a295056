// tests/cpp/tbik_verify.cpp -- the reference's acceptance checks
// (runner.cpp:53-214), re-run through the B200 C++ mirror (tbik_b200/tbik.hpp).
//
// This is what a C++ caller of the reference sees after switching includes
// from "tbik/*.hpp" to "tbik_b200/tbik.hpp": the same check bodies, the same
// Rng streams, the same fingerprints.  Prints one line per check and exits
// non-zero on any failure.  Driven by tests/test_gpu_cpp_api.py.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "tbik_b200/tbik.hpp"

using namespace tbik;

namespace {

int failures = 0;

void report(const std::string& name, bool pass, const std::string& detail) {
  std::printf("%s %s %s\n", pass ? "PASS" : "FAIL", name.c_str(), detail.c_str());
  if (!pass) ++failures;
}

// oracle::tree_reduce (oracle.cpp:11-20), restated for the check.
float tree_reduce(const float* v, std::size_t n) {
  if (n == 1) return v[0];
  return tree_reduce(v, n / 2) + tree_reduce(v + n / 2, n - n / 2);
}

// check_kernel_tp_invariance (runner.cpp:53-91) with both leaf kinds.
void check_kernel_tp_invariance(Leaf leaf, const char* tag) {
  const std::vector<int> tp_set = {1, 2, 4, 8};
  const BlockConfig blocks = default_block_config(Dtype::Bf16);
  std::uint64_t diffs = 0;
  for (std::uint64_t seed = 1; seed <= 5; ++seed) {
    Rng ra(seed, 1), rb(seed, 2);
    const Matrix a = matrix_random_normal(ra, 64, 4096, Dtype::Bf16, 0.0f, 1.0f);
    const Matrix b = matrix_random_normal(rb, 4096, 128, Dtype::Bf16, 0.0f, 1.0f);
    Matrix ref;
    for (std::size_t i = 0; i < tp_set.size(); ++i) {
      Matrix out = row_parallel_forward(a, b, DeviceGroup(tp_set[i]), blocks, 8, leaf);
      if (i == 0)
        ref = std::move(out);
      else
        diffs += bit_diff_count(ref, out);
    }
  }
  report(std::string("kernel_tp_invariance_bf16_") + tag, diffs == 0,
         "m=64 k=4096 n=128 seeds=5 bit_diff_count=" + std::to_string(diffs));
}

void check_config1_golden() {
  Rng ra(1, 1), rb(1, 2);
  const Matrix a = matrix_random_normal(ra, 64, 4096, Dtype::Bf16, 0.0f, 1.0f);
  const Matrix b = matrix_random_normal(rb, 4096, 4096, Dtype::Bf16, 0.0f, 1.0f);
  bool ok = true;
  std::string fps;
  for (int tp : {1, 2, 4, 8}) {
    const std::uint64_t fp =
        bit_fingerprint(row_parallel_forward(a, b, DeviceGroup(tp), default_block_config(Dtype::Bf16), 8, Leaf::Fma));
    char buf[32];
    std::snprintf(buf, sizeof(buf), "%016llx ", static_cast<unsigned long long>(fp));
    fps += buf;
    ok = ok && fp == 0xee480219de506f56ull;  // golden, SURVEY Appendix B
  }
  report("config1_golden_fingerprint_fma_leaf", ok, fps);
}

// check_collective_symmetry (runner.cpp:129-170).
void check_collective_symmetry() {
  std::uint64_t diffs = 0;
  for (int w : {1, 2, 4, 8}) {
    DeviceGroup group(w);
    for (std::uint64_t seed = 1; seed <= 8; ++seed) {
      std::vector<Matrix> contributions;
      for (int r = 0; r < w; ++r) {
        Rng rng(seed, static_cast<std::uint64_t>(r) + 1000 * w);
        contributions.push_back(matrix_random_normal(rng, 1, 8, Dtype::F32, 0.0f, 1.0f));
      }
      const std::vector<Matrix> per_rank = tree_all_reduce_per_rank(group, contributions);
      std::vector<float> leaves(static_cast<std::size_t>(w));
      for (std::int64_t e = 0; e < 8; ++e) {
        for (int r = 0; r < w; ++r) leaves[static_cast<std::size_t>(r)] = contributions[r].at(0, e);
        if (!f32_bit_equal(tree_reduce(leaves.data(), leaves.size()), per_rank[0].at(0, e))) ++diffs;
      }
    }
  }
  report("collective_rank_symmetry", diffs == 0, "bit_diff_count=" + std::to_string(diffs));
}

void check_column_parallel() {
  Rng ra(3, 1), rb(3, 2);
  const Matrix a = matrix_random_normal(ra, 8, 512, Dtype::Bf16, 0.0f, 1.0f);
  const Matrix b = matrix_random_normal(rb, 512, 512, Dtype::Bf16, 0.0f, 1.0f);
  BlockConfig cfg = default_block_config(Dtype::Bf16);
  cfg.block_k = 64;
  const Matrix c1 = column_parallel_forward(a, b, DeviceGroup(1), cfg);
  bool ok = true;
  for (int tp : {2, 4, 8}) ok = ok && bit_equal(c1, column_parallel_forward(a, b, DeviceGroup(tp), cfg));
  bool threw = false;
  try {
    make_column_shard_plan(512, 3);
  } catch (const TbikError& e) {
    threw = e.code() == ErrorCode::ShardError;
  }
  report("column_parallel_invariance", ok && threw, "M=8 K=512 N=512 (SPEC parallel_layers example)");
}

void check_spec_kats() {
  // [1e8, 1, -1e8, 1] -> tree 0 at C = 1/2/4
  const Matrix a = Matrix::from_f32(1, 4, {1e8f, 1.0f, -1e8f, 1.0f});
  const Matrix b = Matrix::from_f32(4, 1, {1.0f, 1.0f, 1.0f, 1.0f});
  bool ok = true;
  for (int tp : {1, 2, 4}) ok = ok && row_parallel_forward(a, b, DeviceGroup(tp), BlockConfig{1, 1, 1, 1}, 4, Leaf::Fma).at(0, 0) == 0.0f;
  const ReductionPlan p = plan_blocks(6144, BlockConfig{64, 256, 128, 0}, 8);
  ok = ok && p.tiles_total == 24 && p.k_first == 3 && p.leaves == 8 && p.depth == 4;
  bool infeasible = false, badworld = false;
  try {
    plan_blocks(4096, BlockConfig{64, 256, 128, 0}, 32);
  } catch (const TbikError& e) {
    infeasible = e.code() == ErrorCode::PlanInfeasible;
  }
  try {
    DeviceGroup g(3);
  } catch (const TbikError& e) {
    badworld = e.code() == ErrorCode::BadWorldSize;
  }
  report("spec_known_answers", ok && infeasible && badworld, "toy tree=0, K=6144 plan, error codes");
}

void check_rmsnorm() {
  Rng rx(11, 1), rg(11, 2);
  const Matrix x = matrix_random_normal(rx, 8, 4096, Dtype::Bf16, 0.0f, 1.0f);
  const Matrix g = matrix_random_normal(rg, 1, 4096, Dtype::F32, 1.0f, 0.02f);
  const Matrix y = rmsnorm(x, g.f32_data(), 1e-5f);
  const Matrix y1 = rmsnorm(x.slice_rows(3, 4), g.f32_data(), 1e-5f);
  bool ok = true;
  for (std::int64_t j = 0; j < 4096; ++j) ok = ok && f32_bit_equal(y.at(3, j), y1.at(0, j));
  report("tree_rmsnorm_batch_invariance", ok, "8x4096 bf16");
}

}  // namespace

int main() {
  try {
    check_kernel_tp_invariance(Leaf::Fma, "fma_leaf");
    check_kernel_tp_invariance(Leaf::Tcgen05, "tcgen05_leaf");
    check_config1_golden();
    check_collective_symmetry();
    check_column_parallel();
    check_spec_kats();
    check_rmsnorm();
  } catch (const TbikError& e) {
    std::printf("FAIL exception %s (status %d)\n", e.what(), e.status());
    return 2;  // tbik_main.cpp:200-203 maps TbikError to exit 2
  }
  std::printf("%s %d failures\n", failures ? "SOME FAILED" : "ALL PASS", failures);
  return failures ? 1 : 0;
}
