// SPDX-License-Identifier: Apache-2.0
// Device-side pieces shared by the fused GAT kernels (gat.cu, gat_lean.cu): work-item
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

// Fast-mode destination record: per head k the float4 {A_r[v,k], lse[v,k], c[v,k], 0}
// (4h floats per row), so one 16-byte load gives an (edge, head) pair all it needs.
__host__ __device__ __forceinline__ int rec_stride(int h) { return 4 * h; }

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
  const uint16_t* lp;    // bf16 copy of the gathered table (Ht for K2, dOut for K4f), or null
  const uint16_t* lp_x;  // K4f bf16 mode: bf16 Ht (the own row, as the forward aggregated it)
  float* part;  // split-row partials
  int64_t row_base, num_local;
  const float* rec;  // fast mode: destination record, float4 {A_r, lse, c, 0} per head (rec_stride)
  int fast;  // K4 fused with K3: dA_r accumulated atomically, its LP term added by gat_lp_dar_kernel
  unsigned* ctr;  // dynamic item fetch (DYN kernels): zeroed work counter in the workspace
  int batch;      // items taken per counter request
  unsigned long long* cnt;  // cost counters of this kernel kind (gnncg_cost_counters), or null
  L2Window win;             // launch attribute only: L2-persisting rows of the gathered table
};

// Cost counters (gnncg_cost_counters; "measured == predicted"): per work item
// the warp adds the edges it walks, and one completed row for an unsplit item (the split-row
// merge kernels add theirs), so the host can check that every edge was aggregated exactly
// once and every row written once (split rows, the work counter's batches) and derive the
// measured flops / io units from the kernel's fixed per-edge and per-row work.
__device__ __forceinline__ void count_item(const GatParams& p, const Item& it, int lane) {
  if (p.cnt != nullptr && lane == 0) {
    atomicAdd(p.cnt, (unsigned long long)(it.e1 - it.e0));
    if (!it.split) atomicAdd(p.cnt + 1, 1ull);
  }
}

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
// per-warp gathers (U rows in flight).  32 warps/SM at <= 64 registers with half the depth
// measured slower at the Reddit shape and is no longer built.
template <int NV, int OCC = 2>
struct GatherDepth {
  static constexpr int U = NV <= 2 ? 8 : (NV == 4 ? 4 : 2);
};

// Lane -> column mapping.  Default: vector i of lane l covers columns [(32 i + l) VW, +VW).
// Paired (pl = lanes per head P > 0; rows that fill the warp exactly, hf = 32 NV VW): lane l
// owns the SAME VW columns of the NV consecutive heads NV (l / P) + i, so the per-head values a
// lane ends up with after K4f's transpose-reduction are adjacent in memory (one vector
// reduction into dA_r); every load instruction still covers whole 128-byte lines.
template <int VW, int NV>
struct Cols {
  int col[NV], hd[NV];
  bool ok[NV];
  __device__ __forceinline__ Cols(int lane, int hf, int f, int pl = 0) {
    if (pl > 0) {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        hd[i] = NV * (lane / pl) + i;
        col[i] = hd[i] * f + (lane % pl) * VW;
        ok[i] = true;
      }
    } else {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        col[i] = (i * 32 + lane) * VW;
        ok[i] = col[i] < hf;
        hd[i] = ok[i] ? col[i] / f : 0;
      }
    }
  }
};

// The paired mapping applies when the row fills the warp exactly and a head spans P = f / VW
// lanes with P dividing 32: returns P, or 0.
__host__ __device__ __forceinline__ int pair_lanes(int h, int f, int VW, int NV) {
  if (h * f != 32 * NV * VW || f % VW != 0) return 0;
  const int P = f / VW;
  return (P >= 1 && P <= 32 && 32 % P == 0) ? P : 0;
}

template <int VW, int NV>
__device__ __forceinline__ void zero(Vec<VW> (&v)[NV]) {
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int q = 0; q < VW; ++q) v[i].x[q] = 0.f;
}

// Gather row `r` of a row-major [*, hf] matrix at this lane's columns.  The address is
// (base + column) + r * row_bytes with a 32 x 32 -> 64-bit multiply-add (one IMAD.WIDE.U32 per
// vector; base + column is loop-invariant), which holds for tables of any size (C5: 5 GB).
template <int VW, int NV>
__device__ __forceinline__ void gather_row(const float* __restrict__ base, uint32_t r, int hf, const Cols<VW, NV>& c,
                                           Vec<VW> (&x)[NV]) {
  // Lanes past the last column load column 0 instead (branch-free); their accumulators are
  // never stored and their partial dots only reach head groups that are masked by `ok`.
  const uint64_t off = (uint64_t)r * (uint32_t)(hf * 4);
#pragma unroll
  for (int i = 0; i < NV; ++i)
    x[i] = ldg_vec<VW>(reinterpret_cast<const float*>(reinterpret_cast<const char*>(base + (c.ok[i] ? c.col[i] : 0)) + off));
}


// Gathered-row storage of one lane vector (VW consecutive columns): fp32, or bf16 kept packed
// in VW/2 registers until it is consumed (LP = the low-precision gather table of
// gnncg_gat_fwd_bf16 / gnncg_gat_bwd_src_fused_bf16; all arithmetic stays fp32).
template <int VW, bool LP>
struct Row;
template <int VW>
struct Row<VW, false> {
  Vec<VW> v;
  __device__ __forceinline__ float operator[](int q) const { return v.x[q]; }
};
template <int VW>
struct Row<VW, true> {
  static_assert(VW % 2 == 0, "bf16 rows need an even lane width");
  uint32_t w[VW / 2];
  // little-endian pairs: element 2j in the low half-word, 2j+1 in the high one
  __device__ __forceinline__ float operator[](int q) const {
    return __uint_as_float((q & 1) ? (w[q >> 1] & 0xffff0000u) : (w[q >> 1] << 16));
  }
};

// gather_row for either storage: `base` is the fp32 or the bf16 table (row stride hf elements).
template <int VW, int NV, bool LP>
__device__ __forceinline__ void gather_rows(const void* __restrict__ base, uint32_t r, int hf, const Cols<VW, NV>& c,
                                            Row<VW, LP> (&x)[NV]) {
  if constexpr (!LP) {
    Vec<VW> t[NV];
    gather_row<VW, NV>(static_cast<const float*>(base), r, hf, c, t);
#pragma unroll
    for (int i = 0; i < NV; ++i) x[i].v = t[i];
  } else {
    const uint64_t off = (uint64_t)r * (uint32_t)(hf * 2);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const char* p = static_cast<const char*>(base) + (c.ok[i] ? c.col[i] : 0) * 2 + off;
      if constexpr (VW == 8) {
        const uint4 t = __ldg(reinterpret_cast<const uint4*>(p));
        x[i].w[0] = t.x; x[i].w[1] = t.y; x[i].w[2] = t.z; x[i].w[3] = t.w;
      } else if constexpr (VW == 4) {
        const uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
        x[i].w[0] = t.x; x[i].w[1] = t.y;
      } else {
        x[i].w[0] = __ldg(reinterpret_cast<const uint32_t*>(p));
      }
    }
  }
}

// Rows in flight per warp for the bf16 table: the same ~64 registers of row data as the fp32
// kernels (GatherDepth), i.e. twice the rows.
template <int VW, int NV>
struct LpDepth {
  static constexpr int R = 128 / (NV * VW);
  static constexpr int U = R > 16 ? 16 : (R < 1 ? 1 : R);
};

}  // namespace gat

// Wavefront-lean K4f (gat_lean.cu): false when the shape is not one it takes.
namespace gat {
bool lean_supported(int h, int f);
bool launch_bwd_src_lean(const GatParams& p, unsigned grid, cudaStream_t s);
bool launch_fwd_lean(const GatParams& p, unsigned grid, cudaStream_t s);
bool launch_fwd_lean_lp(const GatParams& p, cudaStream_t s);
bool launch_bwd_src_lean_lp(const GatParams& p, cudaStream_t s);
}  // namespace gat
}  // namespace gnncg_b200
