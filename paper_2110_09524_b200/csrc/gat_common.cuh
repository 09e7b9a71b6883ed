// SPDX-License-Identifier: Apache-2.0
// Device-side pieces shared by the fused GAT kernels (gat.cu, gat_tma.cu): work-item
// decoding, per-warp tables, lane/column mapping, split-row partial strides.
#pragma once

#include <cfloat>

#include "common.cuh"

namespace gnncg_b200 {
namespace gat {

constexpr int MAXH = 8;          // compiled head limit
constexpr int TS = MAXH + 1;     // padded row of the per-warp edge tables (bank-conflict free)
constexpr int WARPS = 8;         // warps per CTA
constexpr int THREADS = WARPS * kWarp;

struct WarpSmem {
  uint32_t nb[kWarp];
  float t0[kWarp * TS];
  float t1[kWarp * TS];
  float t2[kWarp * TS];
  float red[8 * kWarp];
  float stat[4][MAXH];
};

// Split-row partial records are padded to 16 bytes (vector stores).
__host__ __device__ __forceinline__ int64_t fwd_stride(int h, int f) { return (h * f + 2 * h + 3) / 4 * 4; }
__host__ __device__ __forceinline__ int64_t src_stride(int h, int f) { return (h * f + h + 3) / 4 * 4; }

// Fast-mode destination record {A_r | lse | c}: 3h floats padded to 16 bytes.
__host__ __device__ __forceinline__ int rec_stride(int h) { return (3 * h + 3) / 4 * 4; }

struct Item {
  uint32_t row;
  uint64_t e0, e1;
  bool split;
};

__device__ __forceinline__ Item decode_item(const uint32_t* __restrict__ items, const uint64_t* __restrict__ off,
                                            int64_t wi, int64_t num_split_items, int chunk) {
  Item it;
  it.row = __ldg(items + 2 * wi);
  const uint32_t ch = __ldg(items + 2 * wi + 1);
  const uint64_t rb = __ldg(off + it.row), re = __ldg(off + it.row + 1);
  it.e0 = rb + (uint64_t)ch * (uint64_t)chunk;
  it.e1 = min(re, it.e0 + (uint64_t)chunk);
  it.split = wi < num_split_items;
  return it;
}

// h per-vertex values p[0..h) into registers (vectorised when possible).
__device__ __forceinline__ void load_heads(const float* __restrict__ p, int h, float (&v)[MAXH]) {
  if (h == 8) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    const float4 b = __ldg(reinterpret_cast<const float4*>(p + 4));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else if (h == 4) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
#pragma unroll
    for (int k = 4; k < MAXH; ++k) v[k] = 0.f;
  } else {
#pragma unroll
    for (int k = 0; k < MAXH; ++k) v[k] = k < h ? __ldg(p + k) : 0.f;
  }
}

// Sum, for head `k`, of red[] entries belonging to that head (vector index
// range [k*f/VW, (k+1)*f/VW) of the flattened lane-vector numbering).
template <int VW>
__device__ __forceinline__ float head_sum(const float* red, int k, int f) {
  const int per = f / VW;
  float s = 0.f;
  for (int q = k * per; q < (k + 1) * per; ++q) s += red[q];
  return s;
}

struct GatParams {
  const uint64_t* off;
  const uint32_t* nbr;
  const uint32_t* items;
  int64_t num_items, num_split_items;
  int chunk, h, f;
  float slope;
  const float *Ht, *Al, *Ar, *m, *d, *c, *dOut, *dAr, *a_l, *a_r;
  float *out, *mo, *dd, *co, *dAro, *dHt, *dAl;
  float* part;  // split-row partials
  int64_t row_base, num_local;
  const float* rec;  // fast mode: packed destination record {A_r | lse | c}, stride rec_stride(h)
  int fast;  // K4 fused with K3: dA_r accumulated atomically, its LP term added by gat_lp_dar_kernel
  int64_t hot_rows;  // L2 hint for the neighbour-row gathers (L2Hint; < 0 = off)
};

// ---------------------------------------------------------------------------
// Shared pieces of the three fused kernels.
//
// Per work item the warp walks its edges in 32-edge blocks.  Latency hiding:
//   * neighbour ids are prefetched two blocks ahead and the per-edge logits one
//     block ahead, so the dependent id -> logit loads overlap the previous
//     block's gathers;
//   * the column phase gathers U rows per step (U * NV * VW floats per lane in
//     flight) before consuming any of them.
// ---------------------------------------------------------------------------
// OCC = CTAs per SM the kernel is built for (launch bound): 2 -> 16 warps/SM with deep
// per-warp gathers; 4 -> 32 warps/SM (<= 64 registers) with shallower ones.  More warps
// win for Zipf-distributed gathers (scripts/gather_bench.cu: 9 -> 16 TB/s from 16 to 32
// warps/SM at equal bytes in flight).
template <int NV, int OCC = 2>
struct GatherDepth {
  static constexpr int U = OCC >= 4 ? (NV <= 2 ? 4 : (NV == 4 ? 2 : 1)) : (NV <= 2 ? 8 : (NV == 4 ? 4 : 2));
};

// Runtime choice of OCC (GNNCG_GAT_OCC=2|4, default 2: measured faster at the Reddit shape).
int gat_occupancy();

template <int VW, int NV>
struct Cols {
  int col[NV], hd[NV];
  bool ok[NV];
  __device__ __forceinline__ Cols(int lane, int hf, int f) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      col[i] = (i * 32 + lane) * VW;
      ok[i] = col[i] < hf;
      hd[i] = ok[i] ? col[i] / f : 0;
    }
  }
};

template <int VW, int NV>
__device__ __forceinline__ void zero(Vec<VW> (&v)[NV]) {
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int q = 0; q < VW; ++q) v[i].x[q] = 0.f;
}

// Gather row `r` of a row-major [*, hf] matrix at this lane's columns.
template <int VW, int NV>
__device__ __forceinline__ void gather_row(const float* __restrict__ base, int64_t r, int hf, const Cols<VW, NV>& c,
                                           Vec<VW> (&x)[NV]) {
  // Lanes past the last column load column 0 instead (branch-free); their accumulators are
  // never stored and their partial dots only reach head groups that are masked by `ok`.
  const float* row = base + r * hf;
#pragma unroll
  for (int i = 0; i < NV; ++i) x[i] = ldg_vec<VW>(row + (c.ok[i] ? c.col[i] : 0));
}

// L2 residency hint for the neighbour-row gathers: rows [0, rows) are "hot" and loaded with
// an L2 evict_last policy, the rest with evict_first, so that misses on the long tail do not
// displace the frequently gathered rows.  rows < 0 disables the hints (plain loads).
struct L2Hint {
  int64_t rows;
};

__device__ __forceinline__ L2Hint make_l2_hint(int64_t rows) { return L2Hint{rows}; }

// The policy is created per gathered row (one ALU op) instead of being held in registers.
__device__ __forceinline__ uint64_t l2_policy(bool hot) {
  uint64_t pol;
  if (hot) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

template <int VW>
__device__ __forceinline__ Vec<VW> ldg_vec_pol(const float* p, uint64_t pol) {
  Vec<VW> r;
  if constexpr (VW == 4) {
    asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3])
                 : "l"(p), "l"(pol));
  } else if constexpr (VW == 2) {
    asm("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(r.x[0]), "=f"(r.x[1]) : "l"(p), "l"(pol));
  } else {
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r.x[0]) : "l"(p), "l"(pol));
  }
  return r;
}

template <int VW, int NV>
__device__ __forceinline__ void gather_row(const float* __restrict__ base, int64_t r, int hf, const Cols<VW, NV>& c,
                                           Vec<VW> (&x)[NV], const L2Hint& hint) {
  if (hint.rows < 0) return gather_row<VW, NV>(base, r, hf, c, x);
  const float* row = base + r * hf;
  const uint64_t pol = l2_policy(r < hint.rows);
#pragma unroll
  for (int i = 0; i < NV; ++i) x[i] = ldg_vec_pol<VW>(row + (c.ok[i] ? c.col[i] : 0), pol);
}

// Host side: GNNCG_L2_HOT_ROWS (rows; unset = hints off).
int64_t l2_hot_rows();


}  // namespace gat

// TMA-fed kernels (gat_tma.cu)
namespace gat {
bool tma_fwd_supported(int h, int f);
size_t tma_smem_bytes(int h, int f);
int launch_fwd_tma(const GatParams& p, int* counter, cudaStream_t s);
}  // namespace gat
}  // namespace gnncg_b200
