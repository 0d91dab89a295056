// tbik/demo.hpp -- the hot-path functions of proj/include/tbik/demo.hpp
// (demo.hpp:53-56) on the B200.  The reference's toy decode model
// (DemoConfig / greedy_generate, demo.hpp:18-86) is outside the accelerated path
// (SURVEY.md section 2); its forward template is paper_2511_17826_b200/model.py.
//
//   rmsnorm  TREE-ordered sum of squares (fixed lane chunks + contiguous-halves
//            tree) -- batch- and TP-invariant; within 1e-5 of
//            the reference's sequential rmsnorm (demo.cpp:11-34), not bit-equal.
//   silu     z / (1 + exp(-z)) in f32 with the library's own exp polynomial,
//            identical on every shard and batch; not bit-equal to glibc expf.
#pragma once

#include <vector>

#include "tbik/matrix.hpp"

namespace tbik {

TBIK_CPP_API Matrix rmsnorm(const Matrix& x, const std::vector<float>& gamma, float eps);

TBIK_CPP_API Matrix silu(const Matrix& x);

}  // namespace tbik
