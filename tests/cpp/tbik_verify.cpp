// tests/cpp/tbik_verify.cpp -- the reference's acceptance checks
// (runner.cpp:53-214) against the drop-in headers include/tbik/*.hpp and
// libtbik_b200: a C++ caller of the reference keeps `#include "tbik/layers.hpp"`
// and gets the same Rng streams, the same fingerprints, the same error codes,
// computed on the B200.  (tests/cpp/Makefile also builds the reference's OWN
// runner.cpp against these headers: tests/cpp/ref_verify.)  Prints one line per
// check and exits non-zero on any failure.  Driven by tests/test_gpu_cpp_api.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <set>
#include <string>
#include <vector>

#include "tbik/collective.hpp"
#include "tbik/demo.hpp"
#include "tbik/layers.hpp"
#include "tbik/matmul.hpp"
#include "tbik_b200/peer_group.hpp"

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

// leaf_dot (matmul.hpp:48) on the GPU == the ascending fma chain; the reference's
// leaf-order witness (witness.cpp:53-66): ascending differs from descending at seed 0.
void check_leaf_dot_and_planner_helpers() {
  bool ok = true;
  for (std::uint64_t seed = 0; seed < 4; ++seed) {
    Rng rng(seed, 7);
    std::vector<float> a(8), b(8);
    for (auto& v : a) v = static_cast<float>(rng.next_normal());
    for (auto& v : b) v = static_cast<float>(rng.next_normal());
    float asc = 0.0f, desc = 0.0f;
    for (int k = 0; k < 8; ++k) asc = std::fma(a[k], b[k], asc);
    for (int k = 7; k >= 0; --k) desc = std::fma(a[k], b[k], desc);
    const float got = leaf_dot(a.data(), b.data(), 8);
    ok = ok && f32_bit_equal(got, asc);
    if (seed == 0) ok = ok && !f32_bit_equal(got, desc);
  }
  ok = ok && leaf_dot(nullptr, nullptr, 0) == 0.0f;
  ok = ok && log2_exact(1) == 0 && log2_exact(8) == 3 && log2_exact(9) == 4 && is_power_of_two(64) &&
       !is_power_of_two(0) && !is_power_of_two(12);
  report("leaf_dot_and_planner_helpers", ok, "leaf-order witness seed 0, log2_exact, is_power_of_two");
}

void check_silu() {
  const Matrix x = Matrix::from_f32(1, 6, {-20.0f, -2.0f, -0.5f, 0.0f, 0.75f, 9.0f});
  const Matrix y = silu(x);
  bool ok = y.dtype() == Dtype::F32;
  double worst = 0.0;
  for (int j = 0; j < 6; ++j) {
    const double z = x.at(0, j), want = z / (1.0 + std::exp(-z));
    worst = std::max(worst, std::abs(y.at(0, j) - want) / std::max(std::abs(want), 1e-6));
  }
  ok = ok && worst < 1e-6;
  report("silu", ok, "max rel err vs libm " + std::to_string(worst));
}

// check_baseline_kernel_divergence (runner.cpp:216-237): the status quo gives
// >= 2 distinct bit patterns across TP; the tree path gives exactly one.
void check_baseline_divergence() {
  Rng ra(1, 1), rb(1, 2);
  const Matrix a = matrix_random_normal(ra, 4, 4096, Dtype::F32, 0.0f, 1.0f);
  const Matrix b = matrix_random_normal(rb, 4096, 8, Dtype::F32, 0.0f, 1.0f);
  std::set<std::uint64_t> base, tree;
  for (int tp : {1, 2, 4, 8}) {
    base.insert(bit_fingerprint(baseline_row_parallel_forward(a, b, DeviceGroup(tp))));
    tree.insert(bit_fingerprint(row_parallel_forward(a, b, DeviceGroup(tp), default_block_config(Dtype::F32))));
  }
  const Matrix c1 = baseline_column_parallel_forward(a, b, DeviceGroup(1));
  const bool col_ok = bit_equal(c1, baseline_column_parallel_forward(a, b, DeviceGroup(4)));
  bool shard_err = false;
  try {
    baseline_row_parallel_forward(a.slice_cols(0, 4095), b.slice_rows(0, 4095), DeviceGroup(2));
  } catch (const TbikError& e) {
    shard_err = e.code() == ErrorCode::ShardError;
  }
  report("baseline_kernel_divergence", base.size() >= 2 && tree.size() == 1 && col_ok && shard_err,
         "baseline distinct=" + std::to_string(base.size()) + " tree distinct=" + std::to_string(tree.size()));
}

// DeviceGroup with an explicit rank -> device map, and a one-rank PeerGroup.
void check_groups() {
  Rng ra(5, 1), rb(5, 2);
  const Matrix a = matrix_random_normal(ra, 32, 2048, Dtype::Bf16, 0.0f, 1.0f);
  const Matrix b = matrix_random_normal(rb, 2048, 256, Dtype::Bf16, 0.0f, 1.0f);
  const BlockConfig cfg = default_block_config(Dtype::Bf16);
  const Matrix ref = row_parallel_forward(a, b, DeviceGroup(1), cfg);
  const DeviceGroup g4(4, {0, 0, 0, 0});
  bool ok = g4.device_span() == 1 && bit_equal(ref, row_parallel_forward(a, b, g4, cfg));
  const DeviceGroup g8(8);
  ok = ok && static_cast<int>(g8.devices().size()) == 8 && bit_equal(ref, row_parallel_forward(a, b, g8, cfg));
  PeerGroup pg(1, 0, 0, 32 * 256);
  pg.open_peers(pg.ipc_handle());
  ok = ok && pg.world_size() == 1 && pg.rank() == 0;
  report("device_groups", ok, "explicit device map, DeviceGroup(8) span " + std::to_string(g8.device_span()));
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
    check_leaf_dot_and_planner_helpers();
    check_silu();
    check_baseline_divergence();
    check_groups();
  } catch (const TbikError& e) {
    std::printf("FAIL exception %s (status %d)\n", e.what(), e.status());
    return 2;  // tbik_main.cpp:200-203 maps TbikError to exit 2
  }
  std::printf("%s %d failures\n", failures ? "SOME FAILED" : "ALL PASS", failures);
  return failures ? 1 : 0;
}
