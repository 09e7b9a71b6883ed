// SPDX-License-Identifier: Apache-2.0
// Shared helpers for the sm_100a kernels behind include/gnncg_b200.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "gnncg_b200.h"

namespace gnncg_b200 {

// Thread-local error message behind gnncg_last_error().
void set_error(const char* fmt, ...);
int fail(int status, const char* fmt, ...);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Every compute entry point starts with this: no device => no CPU fallback.
int require_device();

#define GNNCG_CUDA_TRY(expr)                                                                   \
  do {                                                                                         \
    cudaError_t err__ = (expr);                                                                \
    if (err__ != cudaSuccess)                                                                  \
      return ::gnncg_b200::fail(GNNCG_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,     \
                                cudaGetErrorString(err__));                                    \
  } while (0)

// Counts every kernel this library launches (gnncg_launch_count()).
void note_launch();

// L2 access-policy window over the hottest rows of a gathered table (gnncg_l2_persist).
struct L2Window {
  const void* base = nullptr;
  size_t bytes = 0;
};
size_t l2_persist_bytes();
L2Window l2_window(const gnncg_sched_t* sched, const void* table, size_t row_bytes);

// Device cost counters of one kernel kind (gnncg_cost_counters), null when off.
enum CostKind { kCostK2 = 0, kCostK3 = 1, kCostK4 = 2, kCostK4f = 3, kCostLp = 4 };
unsigned long long* cost_slot(int kind);
// slot[0] += a, slot[1] += b on the stream (host-side counts, e.g. the LP rows of K1)
void cost_add(int kind, uint64_t a, uint64_t b, cudaStream_t s);

#define GNNCG_LAUNCH_CHECK()                     \
  do {                                           \
    ::gnncg_b200::note_launch();                 \
    GNNCG_CUDA_TRY(cudaGetLastError());          \
  } while (0)

#define GNNCG_REQUIRE(cond, status, ...)                \
  do {                                                  \
    if (!(cond)) return ::gnncg_b200::fail(status, __VA_ARGS__); \
  } while (0)

#define GNNCG_DEVICE_GUARD()                   \
  do {                                         \
    int rc__ = ::gnncg_b200::require_device(); \
    if (rc__ != GNNCG_OK) return rc__;         \
  } while (0)

constexpr int kWarp = 32;

__device__ __forceinline__ float lrelu(float z, float slope) { return z > 0.f ? z : slope * z; }
__device__ __forceinline__ float lrelu_grad(float z, float slope) { return z > 0.f ? 1.f : slope; }

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Vector of VW consecutive floats (VW in {1,2,4}), read-only path.
template <int VW>
struct Vec {
  float x[VW];
};

template <int VW>
__device__ __forceinline__ Vec<VW> ldg_vec(const float* p) {
  Vec<VW> r;
  if constexpr (VW == 8) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p));
    const float4 u = __ldg(reinterpret_cast<const float4*>(p) + 1);
    r.x[0] = t.x; r.x[1] = t.y; r.x[2] = t.z; r.x[3] = t.w;
    r.x[4] = u.x; r.x[5] = u.y; r.x[6] = u.z; r.x[7] = u.w;
  } else if constexpr (VW == 4) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p));
    r.x[0] = t.x; r.x[1] = t.y; r.x[2] = t.z; r.x[3] = t.w;
  } else if constexpr (VW == 2) {
    const float2 t = __ldg(reinterpret_cast<const float2*>(p));
    r.x[0] = t.x; r.x[1] = t.y;
  } else {
    r.x[0] = __ldg(p);
  }
  return r;
}

// Streaming gather of neighbour rows: read-only path without L1 allocation, so the rows
// (used once per edge) do not evict the reusable per-vertex data from L1.
template <int VW>
__device__ __forceinline__ Vec<VW> ldg_stream(const float* p) {
  Vec<VW> r;
  if constexpr (VW == 4) {
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3])
                 : "l"(p));
  } else if constexpr (VW == 2) {
    asm("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(r.x[0]), "=f"(r.x[1]) : "l"(p));
  } else {
    asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r.x[0]) : "l"(p));
  }
  return r;
}

template <int VW>
__device__ __forceinline__ void st_vec(float* p, const Vec<VW>& v) {
  if constexpr (VW == 8) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v.x[0], v.x[1], v.x[2], v.x[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v.x[4], v.x[5], v.x[6], v.x[7]);
  } else if constexpr (VW == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v.x[0], v.x[1], v.x[2], v.x[3]);
  } else if constexpr (VW == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v.x[0], v.x[1]);
  } else {
    *p = v.x[0];
  }
}

// Ampere-style asynchronous global -> shared copies (L1-allocating: per-vertex values of hub
// vertices are reused).
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gmem_src) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// *p += v (4 consecutive floats, 16-byte aligned) as one vector reduction (sm_90+).
__device__ __forceinline__ void red_add_v4(float* p, const float4& v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// p[0] += a, p[1] += b as one 8-byte vector reduction (sm_90+; p 8-byte aligned).
__device__ __forceinline__ void red_add_v2(float* p, float a, float b) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}

// (d0, d1) = (a0 * b0 + d0, a1 * b1 + d1): one packed FFMA2 (sm_100; each half rounds exactly
// like fmaf, so results are bitwise those of two fmaf).  A broadcast a0 == a1 compiles to the
// scalar-operand form, so the gather kernels issue half the FMA instructions.
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rd, {%0, %1};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rd;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "+f"(d0), "+f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// acc[q] = fmaf(a, x[q], acc[q]) for q < VW, as VW/2 FFMA2 (bitwise identical).
template <int VW, typename Xs>
__device__ __forceinline__ void axpy_vec(float a, const Xs& x, float* acc) {
  if constexpr (VW % 2 == 0) {
#pragma unroll
    for (int q = 0; q < VW; q += 2) ffma2(acc[q], acc[q + 1], a, a, x[q], x[q + 1]);
  } else {
#pragma unroll
    for (int q = 0; q < VW; ++q) acc[q] = fmaf(a, x[q], acc[q]);
  }
}

// sum_q x[q] y[q] with two interleaved FFMA2 partial sums (even / odd q), then one add.
template <int VW, typename Xs, typename Ys>
__device__ __forceinline__ float dot_vec(const Xs& x, const Ys& y) {
  if constexpr (VW % 2 == 0) {
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int q = 0; q < VW; q += 2) ffma2(s0, s1, x[q], x[q + 1], y[q], y[q + 1]);
    return s0 + s1;
  } else {
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < VW; ++q) s = fmaf(x[q], y[q], s);
    return s;
  }
}

// Optional attention-LP epilogue of the tensor-core GEMM (K1 of the GAT layer; gemm_tc.cu).
struct AttnEpi {
  const float* a_l = nullptr;
  const float* a_r = nullptr;
  float* Al = nullptr;  // null: plain GEMM
  float* Ar = nullptr;
  int h = 0, f = 0;
};

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

}  // namespace gnncg_b200
