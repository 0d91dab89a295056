// tbik_tree.cu -- the fixed-order f32 tree kernels that sit above the leaves:
//
//   * tree_combine: out[e] = T( fold_f(ws[0][e] .. ws[f-1][e]), ... )  over a
//     leaf / subtree workspace ws[X][rows][cols].  fold_f is the reference's
//     level-0 sequential prefix ((0 + P0) + P1) + ... (oracle.cpp:120-133,
//     TileReducer level 0, matmul.cpp:100-125) and T is the contiguous-halves
//     tree (oracle.cpp:11-20), evaluated as the same binary counter the
//     reference kernel uses (merges are new + old, commutative).
//   * tree_all_reduce: Algorithm 2 (collective.cpp:52-92) over W rank
//     partials, R[left] += R[left + 2^(l-1)], per element in registers.
//   * ring_reduce: the labelled non-invariant baseline (collective.cpp:94-106).
//
// All three are HBM/NVLink-bound streaming kernels: coalesced 16-byte loads
// where alignment allows, one element per thread otherwise.
#include "tbik_common.cuh"
#include "tbik_internal.h"

namespace tbik_b200 {

namespace {

constexpr int kMaxTreeLevels = 31;

// Binary-counter evaluation of the contiguous-halves tree over the group
// values g_0 .. g_{L-1} (L a power of two).  Registers only: stack[l] holds
// the pending subtree of 2^l groups.
template <int VEC>
__device__ __forceinline__ void tree_push(float (&stack)[kMaxTreeLevels][VEC], uint32_t count,
                                          float (&v)[VEC]) {
  int l = 0;
  uint32_t c = count;
#pragma unroll 1
  while (c & 1u) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = __fadd_rn(v[i], stack[l][i]);
    c >>= 1;
    ++l;
  }
#pragma unroll
  for (int i = 0; i < VEC; ++i) stack[l][i] = v[i];
}

__global__ void tree_combine_kernel(const float* __restrict__ ws, int64_t X, int64_t fold,
                                    int64_t rows, int64_t cols, int64_t slice, float* __restrict__ out,
                                    int64_t ldo) {
  pdl_trigger();
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const int64_t r = e / cols, c = e - r * cols;
  const int64_t L = X / fold;
  float stack[kMaxTreeLevels][1];
  for (int64_t g = 0; g < L; ++g) {
    float v[1] = {0.0f};
    for (int64_t t = g * fold; t < (g + 1) * fold; ++t) v[0] = __fadd_rn(v[0], ws[t * slice + e]);
    // Canonicalise exactly like the reference (acc = 0 + P); for fold >= 1 the
    // first add above already did it.
    tree_push<1>(stack, static_cast<uint32_t>(g), v);
  }
  // After L = 2^j pushes the whole tree sits at stack[j].
  int j = 0;
  while ((int64_t{1} << j) < L) ++j;
  out[r * ldo + c] = stack[j][0];
}

// Fast path for the common split (fold == 1, X = 2^j <= 8 subtree values, 16-byte
// aligned rows): float4 per thread, all X loads in flight, the contiguous-halves
// tree unrolled -- the same bits as tree_combine_kernel (each value canonicalised
// 0 + v, merges commutative).
template <int X>
__global__ void tree_combine_vec_kernel(const float* __restrict__ ws, int64_t rows, int64_t cols, int64_t slice,
                                        float* __restrict__ out, int64_t ldo) {
  pdl_wait();
  pdl_trigger();
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t cq = cols / 4;
  if (q >= rows * cq) return;
  const int64_t r = q / cq, c = (q - r * cq) * 4;
  float4 v[X];
#pragma unroll
  for (int x = 0; x < X; ++x) v[x] = *reinterpret_cast<const float4*>(ws + x * slice + r * cols + c);
#pragma unroll
  for (int x = 0; x < X; ++x) {
    v[x].x = __fadd_rn(0.0f, v[x].x);
    v[x].y = __fadd_rn(0.0f, v[x].y);
    v[x].z = __fadd_rn(0.0f, v[x].z);
    v[x].w = __fadd_rn(0.0f, v[x].w);
  }
#pragma unroll
  for (int st = 2; st <= X; st <<= 1)
#pragma unroll
    for (int left = 0; left < X; left += st) {
      v[left].x = __fadd_rn(v[left].x, v[left + st / 2].x);
      v[left].y = __fadd_rn(v[left].y, v[left + st / 2].y);
      v[left].z = __fadd_rn(v[left].z, v[left + st / 2].z);
      v[left].w = __fadd_rn(v[left].w, v[left + st / 2].w);
    }
  *reinterpret_cast<float4*>(out + r * ldo + c) = v[0];
}

template <bool RING, bool VEC>
__global__ void allreduce_kernel(const PartPtrs parts, int W, int64_t elems,
                                 float* __restrict__ out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t n4 = VEC ? elems / 4 : 0;
  // Vector body: 16-byte loads from each rank's buffer.
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 r[8];
    const int w = W;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < w) r[k] = reinterpret_cast<const float4*>(parts.p[k])[i];
    if (RING) {
      float4 a = r[0];
#pragma unroll
      for (int k = 1; k < 8; ++k)
        if (k < w) {
          a.x = __fadd_rn(a.x, r[k].x);
          a.y = __fadd_rn(a.y, r[k].y);
          a.z = __fadd_rn(a.z, r[k].z);
          a.w = __fadd_rn(a.w, r[k].w);
        }
      reinterpret_cast<float4*>(out)[i] = a;
    } else {
      // collective.cpp:67-74: for l = 1..log2 W, left step 2^l: R[left] += R[left + 2^(l-1)]
#pragma unroll
      for (int l = 1; l <= 3; ++l) {
        const int st = 1 << l, h = 1 << (l - 1);
#pragma unroll
        for (int left = 0; left < 8; left += st)
          if (left + h < w) {
            r[left].x = __fadd_rn(r[left].x, r[left + h].x);
            r[left].y = __fadd_rn(r[left].y, r[left + h].y);
            r[left].z = __fadd_rn(r[left].z, r[left + h].z);
            r[left].w = __fadd_rn(r[left].w, r[left + h].w);
          }
      }
      reinterpret_cast<float4*>(out)[i] = r[0];
    }
  }
  // Scalar tail.
  for (int64_t e = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < elems;
       e += stride) {
    float r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < W) r[k] = parts.p[k][e];
    if (RING) {
      float a = r[0];
#pragma unroll
      for (int k = 1; k < 8; ++k)
        if (k < W) a = __fadd_rn(a, r[k]);
      out[e] = a;
    } else {
#pragma unroll
      for (int l = 1; l <= 3; ++l) {
        const int st = 1 << l, h = 1 << (l - 1);
#pragma unroll
        for (int left = 0; left < 8; left += st)
          if (left + h < W) r[left] = __fadd_rn(r[left], r[left + h]);
      }
      out[e] = r[0];
    }
  }
}

// General W (power of two up to 64): per element recursive halves in a
// register array.  Used for W > 8 only.
__global__ void allreduce_wide_kernel(const PartPtrs parts, int W, int64_t elems,
                                      float* __restrict__ out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < elems; e += stride) {
    float r[64];
    for (int k = 0; k < W; ++k) r[k] = parts.p[k][e];
    for (int st = 2; st <= W; st <<= 1)
      for (int left = 0; left < W; left += st) r[left] = __fadd_rn(r[left], r[left + st / 2]);
    out[e] = r[0];
  }
}

}  // namespace

tbik_status launch_tree_combine(const float* ws, int64_t X, int64_t fold, int64_t rows, int64_t cols,
                                float* out, int64_t ldo, cudaStream_t stream) {
  if (X < 1 || fold < 1 || X % fold) return set_error(TBIK_BAD_ARGUMENT, "tree_combine: bad fold");
  const int64_t L = X / fold;
  if (L & (L - 1)) return set_error(TBIK_BAD_ARGUMENT, "tree_combine: leaves not a power of two");
  if (L > (int64_t{1} << 30)) return set_error(TBIK_BAD_ARGUMENT, "tree_combine: too many leaves");
  const int64_t n = rows * cols;
  if (n == 0) return TBIK_OK;
  const int threads = 256;
  const bool vec = fold == 1 && (X == 2 || X == 4 || X == 8) && cols % 4 == 0 && ldo % 4 == 0 &&
                   (reinterpret_cast<uintptr_t>(ws) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  if (vec) {
    const int64_t nq = n / 4;
    const unsigned vb = static_cast<unsigned>((nq + threads - 1) / threads);
    // programmatic dependent launch: follows the GEMM that wrote ws
    const auto kern = X == 2 ? tree_combine_vec_kernel<2> : X == 4 ? tree_combine_vec_kernel<4> : tree_combine_vec_kernel<8>;
    TBIK_CUDA(launch_pdl(kern, dim3(vb), dim3(threads), 0, stream, ws, rows, cols, n, out, ldo));
    TBIK_CUDA(cudaGetLastError());
    count_launch();
    return TBIK_OK;
  }
  const int64_t blocks = (n + threads - 1) / threads;
  tree_combine_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(ws, X, fold, rows, cols,
                                                                            rows * cols, out, ldo);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

tbik_status launch_allreduce(const PartPtrs& dev_parts, int W, float* out, int64_t elems,
                             bool ring, bool aligned16, cudaStream_t stream) {
  if (elems == 0) return TBIK_OK;
  const int threads = 256;
  int64_t work = aligned16 ? (elems + 3) / 4 : elems;
  int64_t blocks = (work + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  const unsigned nb = static_cast<unsigned>(blocks);
  if (W <= 8 && aligned16) {
    if (ring)
      allreduce_kernel<true, true><<<nb, threads, 0, stream>>>(dev_parts, W, elems, out);
    else
      allreduce_kernel<false, true><<<nb, threads, 0, stream>>>(dev_parts, W, elems, out);
  } else if (W <= 8) {
    if (ring)
      allreduce_kernel<true, false><<<nb, threads, 0, stream>>>(dev_parts, W, elems, out);
    else
      allreduce_kernel<false, false><<<nb, threads, 0, stream>>>(dev_parts, W, elems, out);
  } else if (!ring && W <= 64) {
    allreduce_wide_kernel<<<nb, threads, 0, stream>>>(dev_parts, W, elems, out);
  } else {
    return set_error(TBIK_BAD_WORLD_SIZE, "all-reduce supports W <= 64 (tree) / 8 (ring)");
  }
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

}  // namespace tbik_b200
