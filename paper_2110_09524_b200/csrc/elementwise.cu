// SPDX-License-Identifier: Apache-2.0
//
// Small vertex-side helpers of the training step:
//   * SGD update  params -= lr * grad        (train_step)
//   * loss = sum of exit-tensor entries, deterministic two-level tree
//   * fill                                    (seed gradient dOut = 1)
#include "common.cuh"

namespace gnncg_b200 {
namespace {

constexpr int kSumBlocks = 296;

__global__ void sgd_kernel(int64_t n, float lr, const float* __restrict__ g, float* __restrict__ p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fmaf(-lr, g[i], p[i]);
}

__global__ void fill_kernel(int64_t n, float v, float* __restrict__ x) {
  const int64_t n4 = n / 4;
  float4* x4 = reinterpret_cast<float4*>(x);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    x4[i] = make_float4(v, v, v, v);
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = v;
}

// Fixed assignment of elements to (block, thread) + fixed tree => bitwise reproducible.
__global__ void sum_partial_kernel(int64_t n, const float* __restrict__ x, double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  if ((reinterpret_cast<uintptr_t>(x) & 15) == 0) {  // 16-byte loads, fixed per-thread order
    const int64_t n4 = n >> 2;
    for (int64_t i = tid; i < n4; i += nt) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(x) + i);
      s += ((double)v.x + (double)v.y) + ((double)v.z + (double)v.w);
    }
    for (int64_t i = (n4 << 2) + tid; i < n; i += nt) s += (double)x[i];
  } else {
    for (int64_t i = tid; i < n; i += nt) s += (double)x[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    part[blockIdx.x] = t;
  }
}

// one warp: lane-strided partial sums, then a fixed xor tree (deterministic; the serial
// single-thread loop over 296 partials took 12 us of dependent loads)
__global__ void sum_final_kernel(int nb, const double* __restrict__ part, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  double t = 0.0;
  for (int b = lane; b < nb; b += 32) t += part[b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (threadIdx.x == 0) *out = (float)t;
}

}  // namespace
}  // namespace gnncg_b200

using namespace gnncg_b200;

extern "C" {

int gnncg_sgd_update(int64_t n, float lr, const float* grad, float* param, void* stream) {
  GNNCG_DEVICE_GUARD();
  if (n == 0) return GNNCG_OK;
  GNNCG_REQUIRE(n > 0 && grad && param, GNNCG_ERR_ARG, "sgd_update: bad argument");
  sgd_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 148 * 8), 256, 0, as_stream(stream)>>>(n, lr, grad,
                                                                                                      param);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

int gnncg_fill(int64_t n, float value, float* x, void* stream) {
  GNNCG_DEVICE_GUARD();
  if (n == 0) return GNNCG_OK;
  GNNCG_REQUIRE(n > 0 && x && ((uintptr_t)x % 16 == 0), GNNCG_ERR_ARG, "fill: bad argument (16B alignment)");
  fill_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 1024), 148 * 8), 256, 0, as_stream(stream)>>>(n, value, x);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

size_t gnncg_sum_workspace(void) { return align_up(kSumBlocks * sizeof(double)); }

int gnncg_sum(int64_t n, const float* x, float* out, void* ws, size_t ws_bytes, void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(n >= 0 && out && (n == 0 || x), GNNCG_ERR_ARG, "sum: bad argument");
  GNNCG_REQUIRE(ws && ws_bytes >= gnncg_sum_workspace(), GNNCG_ERR_WORKSPACE, "sum: workspace too small");
  cudaStream_t s = as_stream(stream);
  double* part = static_cast<double*>(ws);
  sum_partial_kernel<<<kSumBlocks, 256, 0, s>>>(n, x, part);
  GNNCG_LAUNCH_CHECK();
  sum_final_kernel<<<1, 32, 0, s>>>(kSumBlocks, part, out);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

}  // extern "C"
