// SPDX-License-Identifier: Apache-2.0
//
// GAT fused graph region on sm_100a: forward (K2) and the two-pass recompute
// backward (K3 over csr_dst, K4 over csc_src), plus the reorganized attention
// LPs and their parameter gradients.
//
// Semantics follow the reference's specification (the executor that would run
// this region, src/executor.cpp, is absent from the reference):
//   fused region 
//   edge-softmax      RS1 (max) / RS2 (sum)
//   recompute plan    stash m, d (O(|V|)); recompute scores and weights
//   backward rules    PAPER.md:615-662 ; empty rows SPEC.md:213
//
// Unified thread mapping: one warp per work item (a whole
// destination row, or a <= chunk-edge slice of a hub row; see gnncg_sched_t).
// Inside a work item the warp alternates two lane mappings:
//   * edge mapping   -- lane j owns edge j of a 32-edge block: gathers the
//     neighbour id and the h attention logits, evaluates LeakyReLU / exp for all
//     heads, writes the 32 x h edge weights to a per-warp shared-memory table;
//   * column mapping -- lane owns NV vectors of VW consecutive feature columns
//     (coalesced 16-byte loads); walks the 32 edges, gathering the neighbour's
//     feature row and FMA-ing it with the edge weight read from shared memory.
// No per-edge value ever reaches HBM; only O(|V| h) statistics are stashed.
#include <cfloat>

#include "common.cuh"
#include "gat_common.cuh"
#include "gat_internal.h"

#include <cuda_bf16.h>

namespace gnncg_b200 {
namespace {

using namespace gat;

// ---------------------------------------------------------------------------
// K2 (overlapped edge phase): the block-synchronous forward with the edge phase moved
// under the gathers.  At the start of every 32-edge block the warp first issues the loads of
// the block's first U neighbour rows, and only then runs the edge phase (logits -> block
// max -> exp weights); the block's logits were copied to shared memory by cp.async one
// block earlier, so the edge phase waits on nothing but its own shuffles and exps, and those
// overlap the row loads.  Same arithmetic as gat_fwd_kernel (bitwise identical results).
// ---------------------------------------------------------------------------
struct OvlSmem {
  uint32_t nb[kWarp];
  float w[kWarp * TS];    // unnormalised weights exp(s - m) of the current block
  float sum[kWarp * TS];  // per-lane running exp-sum partials
  float sc[MAXH];         // rescale factor exp(m_old - m_new) of the current block
  float m[MAXH];          // running max
  float mnext[MAXH];      // running max after the current edge phase
  float ar[MAXH];         // A_r[v]
  float al[kWarp * 12];   // logits A_l[u] of the next block's edges (cp.async), 48-byte lane stride
};

// Logits A_l[u] (h floats) of this lane's edge -> sm.al (asynchronous; waited for before the
// edge phase that reads them).  Only the issuing lane reads its slot.
__device__ __forceinline__ void ovl_issue_logits(OvlSmem& sm, const float* __restrict__ Al, uint32_t u, bool valid,
                                                 int lane, int h) {
  if (valid) {
    const float* src = Al + (int64_t)u * h;
    float* dst = sm.al + lane * 12;
    if ((h & 3) == 0) {
      for (int k = 0; k < h; k += 4) cp_async16(dst + k, src + k);
    } else {
      for (int k = 0; k < h; ++k) cp_async4(dst + k, src + k);
    }
  }
  cp_async_commit();
}

// Edge phase of one 32-edge block: lane owns edge `lane` (valid if lane < n).  Heads are
// processed together (one vote, interleaved shuffle trees) for instruction-level parallelism.
__device__ __forceinline__ void ovl_edge_phase(OvlSmem& sm, int lane, int n, int h, float slope) {
  constexpr int HB = 4;  // heads per pass (bounds the registers live next to the row loads)
  const bool valid = lane < n;
  const float* al = sm.al + lane * 12;  // idle lanes: stale, masked by `valid`
#pragma unroll
  for (int k0 = 0; k0 < MAXH; k0 += HB) {
    if (k0 < h) {
      float s[HB], mn[HB];
      bool up = false;
#pragma unroll
      for (int k = 0; k < HB; ++k) {
        s[k] = (valid && k0 + k < h) ? lrelu(al[k0 + k] + sm.ar[k0 + k], slope) : -FLT_MAX;
        mn[k] = s[k];
        up |= s[k] > sm.m[k0 + k];
      }
      // the block max is only needed when some lane exceeds a running max
      if (__any_sync(0xffffffffu, up)) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int k = 0; k < HB; ++k) mn[k] = fmaxf(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], o));
#pragma unroll
        for (int k = 0; k < HB; ++k) mn[k] = fmaxf(sm.m[k0 + k], mn[k]);
      } else {
#pragma unroll
        for (int k = 0; k < HB; ++k) mn[k] = sm.m[k0 + k];
      }
#pragma unroll
      for (int k = 0; k < HB; ++k) {
        if (k0 + k < h) {
          const int kk = k0 + k;
          const float sc = __expf(sm.m[kk] - mn[k]);
          const float pk = valid ? __expf(s[k] - mn[k]) : 0.f;
          sm.sum[lane * TS + kk] = fmaf(sm.sum[lane * TS + kk], sc, pk);
          sm.w[lane * TS + kk] = pk;
          if (lane == 0) { sm.sc[kk] = sc; sm.mnext[kk] = mn[k]; }
        }
      }
    }
  }
  __syncwarp();
  if (lane < h) sm.m[lane] = sm.mnext[lane];
  __syncwarp();
}

// U rows in flight per warp, CW warps per CTA, MINB CTAs per SM (register budget).
template <int VW, int NV, int U, int CW, int MINB, bool LP = false, bool DYN = false>
__global__ void __launch_bounds__(CW * kWarp) __maxnreg__(MINB >= 2 ? ((65536 / (MINB * CW * kWarp)) / 8 * 8 > 255 ? 255 : (65536 / (MINB * CW * kWarp)) / 8 * 8) : 255) gat_fwd_ovl_kernel(GatParams p) {
  static_assert(32 % U == 0, "U must divide the 32-edge block");
  __shared__ OvlSmem smem[CW];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  OvlSmem& sm = smem[w];
  const int h = p.h, f = p.f, hf = h * f;
  const float slope = p.slope;
  // persistent warps: a fixed stride over the work items (sorted by decreasing size), so no
  // warp idles until the slowest warp of its CTA finishes
  // (the loop is CTA-uniform -- the compiler keeps the memory descriptor in a uniform register
  // -- but carries no barrier: warps advance independently)
  // DYN: warps pull items from a counter instead (items come largest first, so this is a
  // greedy longest-first assignment; the next index is requested at the start of an item)
  // (one item per request: the batched form of K4f changed this kernel's code generation,
  // 1688 -> 2352 instructions, and cost 0.4 ms on the Reddit shape)
  unsigned nx = DYN && lane == 0 ? atomicAdd(p.ctr, 1u) : 0u;
  for (int64_t g = blockIdx.x; DYN || g * CW < p.num_items; g += gridDim.x) {
  int64_t wi;
  if constexpr (DYN) {
    wi = __shfl_sync(0xffffffffu, nx, 0);
    if (wi >= p.num_items) break;
    if (lane == 0) nx = atomicAdd(p.ctr, 1u);
  } else {
    wi = g * CW + w;
    if (wi >= p.num_items) continue;
  }
  const Item it = decode_item(p.items, p.off, wi, p.num_split_items, p.chunk);
  count_item(p, it, lane);

  if (lane < h) {
    sm.ar[lane] = __ldg(p.Ar + (int64_t)it.row * h + lane);
    sm.m[lane] = -FLT_MAX;
  }
#pragma unroll
  for (int k = 0; k < MAXH; ++k) sm.sum[lane * TS + k] = 0.f;
  const Cols<VW, NV> cols(lane, hf, f);
  Vec<VW> acc[NV];
  zero(acc);

  const uint64_t e0 = it.e0, e1 = it.e1;
  uint32_t u_cur = e0 + lane < e1 ? __ldg(p.nbr + e0 + lane) : 0u;
  uint32_t u_nxt = e0 + 32 + lane < e1 ? __ldg(p.nbr + e0 + 32 + lane) : 0u;
  ovl_issue_logits(sm, p.Al, u_cur, e0 + lane < e1, lane, h);

  for (uint64_t base = e0; base < e1; base += 32) {
    const int n = (int)min((uint64_t)32, e1 - base);
    sm.nb[lane] = u_cur;
    __syncwarp();
    // the block's first U rows go out before the edge phase (rows past n repeat the last
    // valid row; their weights are 0)
    const void* tab = LP ? static_cast<const void*>(p.lp) : static_cast<const void*>(p.Ht);
    Row<VW, LP> x[U][NV];
#pragma unroll
    for (int t = 0; t < U; ++t) gather_rows<VW, NV, LP>(tab, sm.nb[min(t, n - 1)], hf, cols, x[t]);
    cp_async_wait_all();
    ovl_edge_phase(sm, lane, n, h, slope);
    // next block: its logits (asynchronous) and the ids of the block after it
    u_cur = u_nxt;
    if (base + 32 < e1) ovl_issue_logits(sm, p.Al, u_cur, base + 32 + lane < e1, lane, h);
    u_nxt = base + 64 + lane < e1 ? __ldg(p.nbr + base + 64 + lane) : 0u;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const float sc = sm.sc[cols.hd[i]];
#pragma unroll
      for (int q = 0; q < VW; ++q) acc[i].x[q] *= sc;
    }
    int j = 0;
    for (;;) {
#pragma unroll
      for (int t = 0; t < U; ++t)
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const float a = sm.w[(j + t) * TS + cols.hd[i]];  // 0 past n (j + t < 32 always)
#pragma unroll
          for (int q = 0; q < VW; ++q) acc[i].x[q] = fmaf(a, x[t][i][q], acc[i].x[q]);
        }
      j += U;
      if (j >= n) break;
#pragma unroll
      for (int t = 0; t < U; ++t) gather_rows<VW, NV, LP>(tab, sm.nb[min(j + t, n - 1)], hf, cols, x[t]);
    }
    __syncwarp();
  }

  __syncwarp();
  float S = 0.f;  // lane k < h: the exp-sum of head k
#pragma unroll
  for (int k = 0; k < MAXH; ++k) {
    if (k < h) {
      const float t = warp_sum(sm.sum[lane * TS + k]);
      if (lane == k) S = t;
    }
  }
  if (lane < h) sm.sc[lane] = S;
  __syncwarp();
  const float mk = e0 < e1 ? (lane < h ? sm.m[lane] : 0.f) : 0.f;
  if (!it.split) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      if (cols.ok[i]) {
        const float den = sm.sc[cols.hd[i]];
        const float inv = den > 0.f ? 1.f / den : 0.f;
        Vec<VW> o;
#pragma unroll
        for (int q = 0; q < VW; ++q) o.x[q] = acc[i].x[q] * inv;
        st_vec<VW>(p.out + (int64_t)it.row * hf + cols.col[i], o);
      }
    }
    if (lane < h) {
      p.mo[(int64_t)it.row * h + lane] = mk;
      p.dd[(int64_t)it.row * h + lane] = S;
    }
  } else {
    float* part = p.part + wi * fwd_stride(h, f);
#pragma unroll
    for (int i = 0; i < NV; ++i)
      if (cols.ok[i]) st_vec<VW>(part + cols.col[i], acc[i]);
    if (lane < h) {
      part[hf + lane] = mk;
      part[hf + h + lane] = S;
    }
  }
  }  // work items
  __syncwarp();
}

// ---------------------------------------------------------------------------
// K3: backward pass 1 over csr_dst.  Per destination v, alpha recomputed from the
// stash (m, d):  c = <g, sum alpha x_u>,  P = <g, sum gate*alpha x_u>,
// Q = sum gate*alpha,  dA_r = P - c Q  (g = dOut[v]; the softmax weights of a
// row sum to one, so no large cancellation).
// ---------------------------------------------------------------------------
template <int VW, int NV, int OCC>
__global__ void __launch_bounds__(THREADS, NV >= 8 ? 1 : OCC) gat_bwd_dst_kernel(GatParams p) {
  __shared__ WarpSmem smem[WARPS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  WarpSmem& sm = smem[w];
  const int64_t wi = (int64_t)blockIdx.x * WARPS + w;
  if (wi >= p.num_items) return;
  const Item it = decode_item(p.items, p.off, wi, p.num_split_items, p.chunk);
  count_item(p, it, lane);
  const int h = p.h, f = p.f, hf = h * f;
  const float slope = p.slope;
  constexpr int U = GatherDepth<NV, OCC>::U;

  if (lane < h) {
    const int64_t r = (int64_t)it.row * h + lane;
    const float dv = __ldg(p.d + r);
    sm.stat[0][lane] = __ldg(p.Ar + r);
    sm.stat[1][lane] = __ldg(p.m + r);
    sm.stat[2][lane] = dv > 0.f ? 1.f / dv : 0.f;
  }
  float Q[MAXH];
#pragma unroll
  for (int k = 0; k < MAXH; ++k) Q[k] = 0.f;
  const Cols<VW, NV> cols(lane, hf, f);
  Vec<VW> g[NV], y[NV], z[NV];
  gather_row<VW, NV>(p.dOut, it.row, hf, cols, g);
  zero(y);
  zero(z);

  const uint64_t e0 = it.e0, e1 = it.e1;
  uint32_t u_cur = e0 + lane < e1 ? __ldg(p.nbr + e0 + lane) : 0u;
  uint32_t u_nxt = e0 + 32 + lane < e1 ? __ldg(p.nbr + e0 + 32 + lane) : 0u;
  float al[MAXH];
  load_heads(p.Al + (int64_t)u_cur * h, h, al);
  __syncwarp();

  for (uint64_t base = e0; base < e1; base += 32) {
    const int n = (int)min((uint64_t)32, e1 - base);
    if (lane < n) {
#pragma unroll
      for (int k = 0; k < MAXH; ++k) {
        if (k < h) {
          const float zz = al[k] + sm.stat[0][k];
          const float a = __expf(lrelu(zz, slope) - sm.stat[1][k]) * sm.stat[2][k];
          const float ga = lrelu_grad(zz, slope) * a;
          sm.t0[lane * TS + k] = a;
          sm.t1[lane * TS + k] = ga;
          Q[k] += ga;
        }
      }
    }
    sm.nb[lane] = u_cur;
    __syncwarp();
    u_cur = u_nxt;
    if (base + 32 + lane < e1) load_heads(p.Al + (int64_t)u_cur * h, h, al);
    u_nxt = base + 64 + lane < e1 ? __ldg(p.nbr + base + 64 + lane) : 0u;
    int j = 0;
    for (; j + U <= n; j += U) {
      Vec<VW> x[U][NV];
#pragma unroll
      for (int t = 0; t < U; ++t) gather_row<VW, NV>(p.Ht, sm.nb[j + t], hf, cols, x[t]);
#pragma unroll
      for (int t = 0; t < U; ++t)
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const float a = sm.t0[(j + t) * TS + cols.hd[i]], ga = sm.t1[(j + t) * TS + cols.hd[i]];
#pragma unroll
          for (int q = 0; q < VW; ++q) {
            y[i].x[q] = fmaf(a, x[t][i].x[q], y[i].x[q]);
            z[i].x[q] = fmaf(ga, x[t][i].x[q], z[i].x[q]);
          }
        }
    }
    for (; j < n; ++j) {
      Vec<VW> x[NV];
      gather_row<VW, NV>(p.Ht, sm.nb[j], hf, cols, x);
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const float a = sm.t0[j * TS + cols.hd[i]], ga = sm.t1[j * TS + cols.hd[i]];
#pragma unroll
        for (int q = 0; q < VW; ++q) {
          y[i].x[q] = fmaf(a, x[i].x[q], y[i].x[q]);
          z[i].x[q] = fmaf(ga, x[i].x[q], z[i].x[q]);
        }
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int k = 0; k < MAXH; ++k)
    if (k < h) Q[k] = warp_sum(Q[k]);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float cp = 0.f, pp = 0.f;
#pragma unroll
    for (int q = 0; q < VW; ++q) { cp = fmaf(g[i].x[q], y[i].x[q], cp); pp = fmaf(g[i].x[q], z[i].x[q], pp); }
    sm.t0[i * 32 + lane] = cp;  // tables are free now; reuse as reduction scratch
    sm.t1[i * 32 + lane] = pp;
  }
  __syncwarp();
  if (lane < h) {
    const float ck = head_sum<VW>(sm.t0, lane, f), pk = head_sum<VW>(sm.t1, lane, f);
    float qk = 0.f;
#pragma unroll
    for (int k = 0; k < MAXH; ++k)
      if (k == lane) qk = Q[k];
    if (!it.split) {
      p.co[(int64_t)it.row * h + lane] = ck;
      p.dAro[(int64_t)it.row * h + lane] = pk - ck * qk;
    } else {
      float* part = p.part + wi * (int64_t)(3 * h);
      part[lane] = ck;
      part[h + lane] = pk;
      part[2 * h + lane] = qk;
    }
  }
}

// ---------------------------------------------------------------------------
// K4: backward pass 2 over csc_src.  Per source u (global), over out-edges to
// local destinations v, alpha and the gate recomputed:
//   dHt[u]  = sum alpha dOut[v]                      (Aggregate backward)
//   dA_l[u] = sum gate*alpha (dalpha - c[v]),  dalpha = <dOut[v], x_u>
// evaluated per 32-edge block as <x_u, sum_b gate*alpha dOut[v]> - sum_b gate*alpha c[v]
// (out-edge sums are NOT normalised, so the difference is taken block by block to
// avoid cancellation on hub sources), then the LP epilogue
// dHt[u] += dA_l[u] (x) a_l + dA_r[u] (x) a_r.
// ---------------------------------------------------------------------------
template <int VW, int NV, int OCC>
__global__ void __launch_bounds__(THREADS, NV >= 8 ? 1 : OCC) gat_bwd_src_kernel(GatParams p) {
  __shared__ WarpSmem smem[WARPS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  WarpSmem& sm = smem[w];
  const int64_t wi = (int64_t)blockIdx.x * WARPS + w;
  if (wi >= p.num_items) return;
  const Item it = decode_item(p.items, p.off, wi, p.num_split_items, p.chunk);
  count_item(p, it, lane);
  const int h = p.h, f = p.f, hf = h * f;
  const float slope = p.slope;
  const int64_t u = it.row;
  constexpr int U = GatherDepth<NV, OCC>::U;

  if (lane < h) sm.stat[3][lane] = __ldg(p.Al + u * h + lane);
  float dal_acc = 0.f;  // lane k < h: dA_l[u, k]
  const Cols<VW, NV> cols(lane, hf, f);
  Vec<VW> x[NV], acc[NV], wv[NV];
  gather_row<VW, NV>(p.Ht, u, hf, cols, x);
  zero(acc);
  zero(wv);

  const uint64_t e0 = it.e0, e1 = it.e1;
  uint32_t v_cur = e0 + lane < e1 ? __ldg(p.nbr + e0 + lane) : 0u;
  __syncwarp();

  for (uint64_t base = e0; base < e1; base += 32) {
    const int n = (int)min((uint64_t)32, e1 - base);
    if (lane < n) {
      float arv[MAXH], mv[MAXH], dv[MAXH], cv[MAXH];
      load_heads(p.Ar + (int64_t)v_cur * h, h, arv);
      load_heads(p.m + (int64_t)v_cur * h, h, mv);
      load_heads(p.d + (int64_t)v_cur * h, h, dv);
      load_heads(p.c + (int64_t)v_cur * h, h, cv);
#pragma unroll
      for (int k = 0; k < MAXH; ++k) {
        if (k < h) {
          const float zz = sm.stat[3][k] + arv[k];
          const float a = dv[k] > 0.f ? __expf(lrelu(zz, slope) - mv[k]) / dv[k] : 0.f;
          const float ga = lrelu_grad(zz, slope) * a;
          sm.t0[lane * TS + k] = a;
          sm.t1[lane * TS + k] = ga;
          sm.t2[lane * TS + k] = ga * cv[k];
        }
      }
    }
    sm.nb[lane] = v_cur;
    __syncwarp();
    v_cur = base + 32 + lane < e1 ? __ldg(p.nbr + base + 32 + lane) : 0u;
    int j = 0;
    for (; j + U <= n; j += U) {
      Vec<VW> gv[U][NV];
#pragma unroll
      for (int t = 0; t < U; ++t) gather_row<VW, NV>(p.dOut, sm.nb[j + t], hf, cols, gv[t]);
#pragma unroll
      for (int t = 0; t < U; ++t)
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const float a = sm.t0[(j + t) * TS + cols.hd[i]], ga = sm.t1[(j + t) * TS + cols.hd[i]];
#pragma unroll
          for (int q = 0; q < VW; ++q) {
            acc[i].x[q] = fmaf(a, gv[t][i].x[q], acc[i].x[q]);
            wv[i].x[q] = fmaf(ga, gv[t][i].x[q], wv[i].x[q]);
          }
        }
    }
    for (; j < n; ++j) {
      Vec<VW> gv[NV];
      gather_row<VW, NV>(p.dOut, sm.nb[j], hf, cols, gv);
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const float a = sm.t0[j * TS + cols.hd[i]], ga = sm.t1[j * TS + cols.hd[i]];
#pragma unroll
        for (int q = 0; q < VW; ++q) {
          acc[i].x[q] = fmaf(a, gv[i].x[q], acc[i].x[q]);
          wv[i].x[q] = fmaf(ga, gv[i].x[q], wv[i].x[q]);
        }
      }
    }
    // block-level dA_l contribution
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      float s = 0.f;
#pragma unroll
      for (int q = 0; q < VW; ++q) { s = fmaf(x[i].x[q], wv[i].x[q], s); wv[i].x[q] = 0.f; }
      sm.red[i * 32 + lane] = s;
    }
    __syncwarp();
    if (lane < h) {
      float r = head_sum<VW>(sm.red, lane, f);
      for (int jj = 0; jj < n; ++jj) r -= sm.t2[jj * TS + lane];
      dal_acc += r;
    }
    __syncwarp();
  }
  if (lane < h) {
    sm.stat[0][lane] = dal_acc;
    const bool local = u >= p.row_base && u < p.row_base + p.num_local;
    sm.stat[1][lane] = local ? __ldg(p.dAr + (u - p.row_base) * h + lane) : 0.f;
  }
  __syncwarp();
  if (!it.split) {
    if (lane < h) p.dAl[u * h + lane] = sm.stat[0][lane];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      if (cols.ok[i]) {
        const float dal = sm.stat[0][cols.hd[i]], dar = sm.stat[1][cols.hd[i]];
        const Vec<VW> al = ldg_vec<VW>(p.a_l + cols.col[i]);
        const Vec<VW> ar = ldg_vec<VW>(p.a_r + cols.col[i]);
        Vec<VW> o;
#pragma unroll
        for (int q = 0; q < VW; ++q) o.x[q] = acc[i].x[q] + dal * al.x[q] + dar * ar.x[q];
        st_vec<VW>(p.dHt + u * hf + cols.col[i], o);
      }
    }
  } else {
    float* part = p.part + wi * src_stride(h, f);
#pragma unroll
    for (int i = 0; i < NV; ++i)
      if (cols.ok[i]) st_vec<VW>(part + cols.col[i], acc[i]);
    if (lane < h) part[hf + lane] = sm.stat[0][lane];
  }
}

// ---------------------------------------------------------------------------
// K4 "fast" (SPEC.md:378 fast mode): backward pass 2 with pass 1 folded in.
// With c[v] = <dOut[v], out[v]> per head (= sum_e alpha_e dalpha_e, the softmax
// backward identity; gat_rowdot_kernel), a single pass over csc_src computes per
// edge dalpha_e = <dOut[v], x_u> and dz_e = gate*alpha (dalpha_e - c[v]); dA_l[u]
// sums dz_e in the warp, dA_r[v] receives dz_e by a global red (order-
// nondeterministic, tolerance-tested).  Removes K3's whole csr_dst gather pass.
//
// Per-edge head dots without per-edge shuffles: for a group of U gathered edges
// each lane holds U*NV partial dots; a butterfly transpose-reduction over the
// PER lanes that share a head (log2(PER) steps, halving the values each step)
// leaves lane r of every PER-group with the complete dots of (edge, vector)
// pairs [r*NOUT, r*NOUT+NOUT) -- U*NV*(1-1/PER) shuffles instead of U*NV*log2(PER).
// ---------------------------------------------------------------------------
template <int CNT, int OFF>
__device__ __forceinline__ void butterfly(float* v, int lane) {
  if constexpr (OFF >= 1) {
    const bool up = (lane & OFF) != 0;
#pragma unroll
    for (int j = 0; j < CNT / 2; ++j) {
      const float send = up ? v[j] : v[j + CNT / 2];
      const float keep = up ? v[j + CNT / 2] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, OFF);
    }
    butterfly<CNT / 2, OFF / 2>(v, lane);
  }
}

template <int VW, int NV, int PER, int OCC, bool LP = false, bool PAIR = false, bool DYN = false>
__global__ void __launch_bounds__(THREADS, NV >= 8 ? 1 : OCC) gat_bwd_src_fast_kernel(GatParams p) {
  constexpr int U = LP ? LpDepth<VW, NV>::U : GatherDepth<NV, OCC>::U;
  // next-group loads issued per half-group: bf16 rows only (packed rows leave the registers for
  // it; in fp32 the extra live rows spill -- measured 8.78 -> 8.64 ms bf16, 11.8 -> 16.1 ms fp32)
  constexpr bool HALVES = LP && NV == 1 && U >= 2 && U % 2 == 0;
  constexpr int NVAL = U * NV, NOUT = NVAL / PER;
  static_assert(NVAL % PER == 0, "fast K4 needs U*NV to be a multiple of the lanes per head");
  __shared__ WarpSmem smem[WARPS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  WarpSmem& sm = smem[w];
  const int h = p.h, f = p.f, hf = h * f;
  const float slope = p.slope;
  const int r = lane & (PER - 1);  // rank inside the head's lane group
  // persistent CTA-uniform item loop (as in gat_fwd_ovl_kernel), no barrier inside
  // as in gat_fwd_ovl_kernel, but p.batch items per request when items are short (C5: one
  // counter address serves ~10^8 requests per second)
  unsigned nx = DYN && lane == 0 ? atomicAdd(p.ctr, (unsigned)p.batch) : 0u;
  int64_t cur = 0, cend = 0;
  for (int64_t g = blockIdx.x; DYN || g * WARPS < p.num_items; g += gridDim.x) {
  int64_t wi;
  if constexpr (DYN) {
    if (cur >= cend) {
      cur = __shfl_sync(0xffffffffu, nx, 0);
      cend = cur + p.batch;
      if (lane == 0) nx = atomicAdd(p.ctr, (unsigned)p.batch);
    }
    wi = cur++;
    if (wi >= p.num_items) break;
  } else {
    wi = g * WARPS + w;
    if (wi >= p.num_items) continue;
  }
  const Item it = decode_item(p.items, p.off, wi, p.num_split_items, p.chunk);
  count_item(p, it, lane);
  const int64_t u = it.row;

  if (lane < h) sm.stat[3][lane] = __ldg(p.Al + u * h + lane);
  // PAIR: lane's vectors in adjacent heads -> after the transpose-reduction a lane holds one
  // edge's dz for heads (2g, 2g+1): one 8-byte reduction into dA_r instead of two
  static_assert(!PAIR || (NV == 2 && NOUT == 2), "paired reductions: two vectors, two outputs per lane");
  const Cols<VW, NV> cols(lane, hf, f, PAIR ? PER : 0);
  Vec<VW> x[NV], acc[NV];
  float dal[NV];
  if constexpr (LP) {
    // bf16 mode: the own row is the same rounded Ht[u] the forward aggregated, so that
    // sum_e alpha_e dalpha_e = <dOut~[v], out[v]> = c[v] holds exactly as in fp32 mode
    Row<VW, true> xr[NV];
    gather_rows<VW, NV, true>(p.lp_x, (uint32_t)u, hf, cols, xr);
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int q = 0; q < VW; ++q) x[i].x[q] = xr[i][q];
  } else {
    gather_row<VW, NV>(p.Ht, u, hf, cols, x);
  }
  zero(acc);
#pragma unroll
  for (int i = 0; i < NV; ++i) dal[i] = 0.f;

  const uint64_t e0 = it.e0, e1 = it.e1;
  uint32_t v_cur = e0 + lane < e1 ? __ldg(p.nbr + e0 + lane) : 0u;
  __syncwarp();

  const void* tab = LP ? static_cast<const void*>(p.lp) : static_cast<const void*>(p.dOut);
  for (uint64_t base = e0; base < e1; base += 32) {
    const int n = (int)min((uint64_t)32, e1 - base);
    sm.nb[lane] = v_cur;  // idle lanes hold row 0: a valid row whose weights are 0
    __syncwarp();
    // the first half of the block's first row group goes out before the dependent record
    // loads of the edge phase (the whole group would not fit next to the records' registers)
    constexpr int UH = U >= 2 ? U / 2 : 1;
    Row<VW, LP> gv[U][NV];
#pragma unroll
    for (int t = 0; t < UH; ++t) gather_rows<VW, NV, LP>(tab, sm.nb[t], hf, cols, gv[t]);
    {
      const bool valid = lane < n;
      // packed destination record {A_r | lse = m + log d | c} (gat_bwd_prep_kernel): one
      // contiguous 3h-float read per edge, and alpha = exp(s - lse) needs no divide
      const float4* rec = reinterpret_cast<const float4*>(p.rec + (int64_t)v_cur * rec_stride(h));
      float arv[MAXH], lse[MAXH], cv[MAXH];
#pragma unroll
      for (int k = 0; k < MAXH; ++k) {
        const float4 q = k < h ? __ldg(rec + k) : make_float4(0.f, 0.f, 0.f, 0.f);
        arv[k] = q.x; lse[k] = q.y; cv[k] = q.z;
      }
#pragma unroll
      for (int k = 0; k < MAXH; ++k) {
        if (k < h) {
          const float zz = sm.stat[3][k] + arv[k];
          const float a = valid ? __expf(lrelu(zz, slope) - lse[k]) : 0.f;
          sm.t0[lane * TS + k] = a;
          sm.t1[lane * TS + k] = lrelu_grad(zz, slope) * a;
          sm.t2[lane * TS + k] = cv[k];
        }
      }
    }
    __syncwarp();
    v_cur = base + 32 + lane < e1 ? __ldg(p.nbr + base + 32 + lane) : 0u;
#pragma unroll
    for (int t = UH; t < U; ++t) gather_rows<VW, NV, LP>(tab, sm.nb[t], hf, cols, gv[t]);
    for (int j = 0;;) {
      float pd[NVAL];
      // two half-groups: once the first half's rows are consumed, its registers take the next
      // group's first half (in flight during the second half's FMAs, the butterfly and the
      // reductions) -- the heavy per-row work (weights + dots) no longer leaves the warp idle
      const bool more = j + U < n;
#pragma unroll
      for (int hg = 0; hg < 2; ++hg) {
#pragma unroll
        for (int t = hg * (U / 2); t < (hg + 1) * (U / 2); ++t) {
          const int e = (j + t) & 31;
#pragma unroll
          for (int i = 0; i < NV; ++i) {
            const float a = sm.t0[e * TS + cols.hd[i]];
            axpy_vec<VW>(a, gv[t][i], acc[i].x);
            pd[t * NV + i] = dot_vec<VW>(x[i].x, gv[t][i]);
          }
        }
        if (HALVES && more) {
#pragma unroll
          for (int t = hg * (U / 2); t < (hg + 1) * (U / 2); ++t)
            gather_rows<VW, NV, LP>(tab, sm.nb[(j + U + t) & 31], hf, cols, gv[t]);
        }
      }
      butterfly<NVAL, PER / 2>(pd, lane);
      float dzp[NOUT];
#pragma unroll
      for (int q = 0; q < NOUT; ++q) {
        const int idx = r * NOUT + q;
        const int t = idx / NV, i = idx % NV;
        int hd = cols.hd[0];
        bool ok = cols.ok[0];
#pragma unroll
        for (int ii = 1; ii < NV; ++ii)
          if (i == ii) { hd = cols.hd[ii]; ok = cols.ok[ii]; }
        const int e = j + t;
        const bool valid = ok && e < n;
        const float dz = valid ? sm.t1[e * TS + hd] * (pd[q] - sm.t2[e * TS + hd]) : 0.f;
#pragma unroll
        for (int ii = 0; ii < NV; ++ii)
          if (i == ii) dal[ii] += dz;
        dzp[q] = dz;
        if (!PAIR && valid) atomicAdd(p.dAro + (int64_t)sm.nb[e] * h + hd, dz);
      }
      if constexpr (PAIR) {
        // both outputs belong to edge r of the group, heads hd[0], hd[0] + 1; the lane group
        // with the next two heads of the same edge is 8 lanes up: even groups collect them and
        // add four adjacent heads at once (16-byte aligned: hd[0] = 4 g')
        const float o0 = __shfl_down_sync(0xffffffffu, dzp[0], PER);
        const float o1 = __shfl_down_sync(0xffffffffu, dzp[1], PER);
        const int e = j + r;
        if (((lane / PER) & 1) == 0 && e < n)
          red_add_v4(p.dAro + (int64_t)sm.nb[e] * h + cols.hd[0], make_float4(dzp[0], dzp[1], o0, o1));
      }
      j += U;
      if (j >= n) break;
      if constexpr (!HALVES) {
#pragma unroll
        for (int t = 0; t < U; ++t) gather_rows<VW, NV, LP>(tab, sm.nb[(j + t) & 31], hf, cols, gv[t]);
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) {
#pragma unroll
    for (int o = 1; o < PER; o <<= 1) dal[i] += __shfl_xor_sync(0xffffffffu, dal[i], o);
    if (cols.ok[i] && r == 0) sm.stat[0][cols.hd[i]] = dal[i];
  }
  __syncwarp();
  if (!it.split) {
    if (lane < h) p.dAl[u * h + lane] = sm.stat[0][lane];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      if (cols.ok[i]) {
        const float dl = sm.stat[0][cols.hd[i]];
        const Vec<VW> al = ldg_vec<VW>(p.a_l + cols.col[i]);
        Vec<VW> o;
#pragma unroll
        for (int q = 0; q < VW; ++q) o.x[q] = fmaf(dl, al.x[q], acc[i].x[q]);
        st_vec<VW>(p.dHt + u * hf + cols.col[i], o);
      }
    }
  } else {
    float* part = p.part + wi * src_stride(h, f);
#pragma unroll
    for (int i = 0; i < NV; ++i)
      if (cols.ok[i]) st_vec<VW>(part + cols.col[i], acc[i]);
    if (lane < h) part[hf + lane] = sm.stat[0][lane];
  }
  __syncwarp();
  }  // work items
}

// Fast-mode input of K4f, per destination v and head k (row-local, vertex tensors only):
//   rec[v, k] = float4 { A_r[v,k], lse[v,k] = m[v,k] + log d[v,k], c[v,k] = <dOut[v,k,:], out[v,k,:]>, 0 }
// c = sum_e alpha_e dalpha_e by the softmax-backward identity; lse folds the stashed
// (m, d) so that alpha_e = exp(s_e - lse).  Empty rows (d = 0) get lse = 0 (never read).
__global__ void gat_bwd_prep_kernel(int64_t rows, int h, int f, const float* __restrict__ dOut,
                                    const float* __restrict__ out, const float* __restrict__ Ar,
                                    const float* __restrict__ m, const float* __restrict__ d,
                                    float* __restrict__ rec) {
  const int rpb = blockDim.x / h;  // rows per block step (h <= blockDim.x): no per-element 64-bit divide
  const int rr = threadIdx.x / h, k = threadIdx.x - rr * h;
  if (rr >= rpb) return;
  const bool vec = (f % 4) == 0;
  const int rs = rec_stride(h);
  for (int64_t v = (int64_t)blockIdx.x * rpb + rr; v < rows; v += (int64_t)gridDim.x * rpb) {
    const int64_t i = v * h + k;
    const float* g = dOut + i * f;
    const float* o = out + i * f;
    float s = 0.f;
    if (vec) {
      for (int j = 0; j < f; j += 4) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(g + j));
        const float4 b = __ldg(reinterpret_cast<const float4*>(o + j));
        s = fmaf(a.x, b.x, s); s = fmaf(a.y, b.y, s); s = fmaf(a.z, b.z, s); s = fmaf(a.w, b.w, s);
      }
    } else {
      for (int j = 0; j < f; ++j) s = fmaf(__ldg(g + j), __ldg(o + j), s);
    }
    const float dv = __ldg(d + i);
    reinterpret_cast<float4*>(rec + v * rs)[k] =
        make_float4(__ldg(Ar + i), dv > 0.f ? __ldg(m + i) + __logf(dv) : 0.f, s, 0.f);
  }
}

// bf16 mode of gat_bwd_prep_kernel: c = <dOut~, out> with dOut~ = bf16(dOut) (the rows K4f
// gathers), and dOut~ written out as the gather table (f % 4 == 0).
__global__ void gat_bwd_prep_bf16_kernel(int64_t rows, int h, int f, const float* __restrict__ dOut,
                                         const float* __restrict__ out, const float* __restrict__ Ar,
                                         const float* __restrict__ m, const float* __restrict__ d,
                                         float* __restrict__ rec, uint16_t* __restrict__ dOut_lp) {
  const int rpb = blockDim.x / h;  // rows per block step (h <= blockDim.x): no per-element 64-bit divide
  const int rr = threadIdx.x / h, k = threadIdx.x - rr * h;
  if (rr >= rpb) return;
  const int rs = rec_stride(h);
  for (int64_t v = (int64_t)blockIdx.x * rpb + rr; v < rows; v += (int64_t)gridDim.x * rpb) {
    const int64_t i = v * h + k;
    const float* g = dOut + i * f;
    const float* o = out + i * f;
    uint2* gl = reinterpret_cast<uint2*>(dOut_lp + i * f);
    float s = 0.f;
    for (int j = 0; j < f; j += 4) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(g + j));
      const float4 b = __ldg(reinterpret_cast<const float4*>(o + j));
      const __nv_bfloat16 ax = __float2bfloat16_rn(a.x), ay = __float2bfloat16_rn(a.y);
      const __nv_bfloat16 az = __float2bfloat16_rn(a.z), aw = __float2bfloat16_rn(a.w);
      s = fmaf(__bfloat162float(ax), b.x, s); s = fmaf(__bfloat162float(ay), b.y, s);
      s = fmaf(__bfloat162float(az), b.z, s); s = fmaf(__bfloat162float(aw), b.w, s);
      gl[j / 4] = make_uint2((uint32_t)__bfloat16_as_ushort(ax) | ((uint32_t)__bfloat16_as_ushort(ay) << 16),
                             (uint32_t)__bfloat16_as_ushort(az) | ((uint32_t)__bfloat16_as_ushort(aw) << 16));
    }
    const float dv = __ldg(d + i);
    reinterpret_cast<float4*>(rec + v * rs)[k] =
        make_float4(__ldg(Ar + i), dv > 0.f ? __ldg(m + i) + __logf(dv) : 0.f, s, 0.f);
  }
}

// dHt[row_base + r, :] += dA_r[r] (x) a_r  for the local rows (fast-mode LP epilogue).
__global__ void gat_lp_dar_kernel(int64_t rows, int64_t row_base, int h, int f, const float* __restrict__ dAr,
                                  const float* __restrict__ a_r, float* __restrict__ dHt) {
  const int hf = h * f;
  if ((f & 3) == 0) {
    // float4 columns (one head each), threads = (row slot, column quad): no 64-bit division
    const int q4 = hf >> 2;
    const int rpb = max(1, (int)blockDim.x / q4);  // rows per block step
    const int slot = threadIdx.x / q4, c4 = threadIdx.x - slot * q4;
    if (slot >= rpb) return;
    const float4 ar = __ldg(reinterpret_cast<const float4*>(a_r) + c4);
    const int k = (c4 * 4) / f;
    for (int64_t r = (int64_t)blockIdx.x * rpb + slot; r < rows; r += (int64_t)gridDim.x * rpb) {
      const float g = __ldg(dAr + r * h + k);
      float4* d = reinterpret_cast<float4*>(dHt + (row_base + r) * hf) + c4;
      float4 v = *d;
      v.x = fmaf(g, ar.x, v.x); v.y = fmaf(g, ar.y, v.y); v.z = fmaf(g, ar.z, v.z); v.w = fmaf(g, ar.w, v.w);
      *d = v;
    }
    return;
  }
  const int64_t n = rows * hf;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / hf;
    const int col = (int)(i % hf);
    dHt[(row_base + r) * hf + col] += __ldg(dAr + r * h + col / f) * __ldg(a_r + col);
  }
}

// Merge of split-row partials (forward): online-softmax combination in chunk order.
__global__ void gat_fwd_merge_kernel(GatParams p, const uint32_t* __restrict__ split_rows,
                                     const uint32_t* __restrict__ split_first, int64_t num_split_rows) {
  __shared__ float st[WARPS][2][MAXH];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t sr = (int64_t)blockIdx.x * WARPS + w;
  if (sr >= num_split_rows) return;
  if (p.cnt != nullptr && lane == 0) atomicAdd(p.cnt + 1, 1ull);  // a split row completed
  const int h = p.h, f = p.f, hf = h * f;
  const int64_t stride = fwd_stride(h, f);
  const uint32_t row = split_rows[sr];
  const int64_t i0 = split_first[sr], i1 = split_first[sr + 1];
  if (lane < h) {
    float mk = -FLT_MAX;
    for (int64_t it = i0; it < i1; ++it) mk = fmaxf(mk, p.part[it * stride + hf + lane]);
    float sk = 0.f;
    for (int64_t it = i0; it < i1; ++it)
      sk += p.part[it * stride + hf + h + lane] * __expf(p.part[it * stride + hf + lane] - mk);
    st[w][0][lane] = mk;
    st[w][1][lane] = sk;
    p.mo[(int64_t)row * h + lane] = mk;
    p.dd[(int64_t)row * h + lane] = sk;
  }
  __syncwarp();
  for (int c = lane; c < hf; c += 32) {
    const int hd = c / f;
    const float mk = st[w][0][hd], sk = st[w][1][hd];
    float s = 0.f;
    for (int64_t it = i0; it < i1; ++it) s += p.part[it * stride + c] * __expf(p.part[it * stride + hf + hd] - mk);
    p.out[(int64_t)row * hf + c] = sk > 0.f ? s / sk : 0.f;
  }
}

__global__ void gat_bwd_dst_merge_kernel(GatParams p, const uint32_t* __restrict__ split_rows,
                                         const uint32_t* __restrict__ split_first, int64_t num_split_rows) {
  const int64_t sr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int h = p.h;
  if (sr >= num_split_rows * h) return;
  const int64_t r = sr / h;
  const int k = (int)(sr % h);
  if (p.cnt != nullptr && k == 0) atomicAdd(p.cnt + 1, 1ull);  // a split row completed
  const uint32_t row = split_rows[r];
  float c = 0.f, P = 0.f, Q = 0.f;
  for (int64_t it = split_first[r]; it < split_first[r + 1]; ++it) {
    c += p.part[it * 3 * h + k];
    P += p.part[it * 3 * h + h + k];
    Q += p.part[it * 3 * h + 2 * h + k];
  }
  p.co[(int64_t)row * h + k] = c;
  p.dAro[(int64_t)row * h + k] = P - c * Q;
}

__global__ void gat_bwd_src_merge_kernel(GatParams p, const uint32_t* __restrict__ split_rows,
                                         const uint32_t* __restrict__ split_first, int64_t num_split_rows) {
  __shared__ float st[WARPS][2][MAXH];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t sr = (int64_t)blockIdx.x * WARPS + w;
  if (sr >= num_split_rows) return;
  if (p.cnt != nullptr && lane == 0) atomicAdd(p.cnt + 1, 1ull);  // a split row completed
  const int h = p.h, f = p.f, hf = h * f;
  const int64_t stride = src_stride(h, f);
  const int64_t u = split_rows[sr];
  const int64_t i0 = split_first[sr], i1 = split_first[sr + 1];
  if (lane < h) {
    float dal = 0.f;
    for (int64_t it = i0; it < i1; ++it) dal += p.part[it * stride + hf + lane];
    st[w][0][lane] = dal;
    const bool local = u >= p.row_base && u < p.row_base + p.num_local;
    st[w][1][lane] = (local && !p.fast) ? p.dAr[(u - p.row_base) * h + lane] : 0.f;
    p.dAl[u * h + lane] = dal;
  }
  __syncwarp();
  for (int c = lane; c < hf; c += 32) {
    const int hd = c / f;
    float s = 0.f;
    for (int64_t it = i0; it < i1; ++it) s += p.part[it * stride + c];
    p.dHt[u * hf + c] = s + st[w][0][hd] * p.a_l[c] + st[w][1][hd] * p.a_r[c];
  }
}

// ---------------------------------------------------------------------------
// Reorganized LPs and their parameter gradients.
// ---------------------------------------------------------------------------
// A_l[v, k] = <Ht[v, k f : (k+1) f], a_l[k]> (A_r likewise), one thread per (row, head), columns
// summed in order (bitwise the same as K1's LP epilogue).  A block covers 256 / h rows at a time
// and strides over rows, so the (row, head) split is one division per thread, not a 64-bit
// divide and modulo per element (which made the kernel ~3x slower than its bytes at C5).
__global__ void attn_dots_kernel(int64_t rows, int h, int f, const float* __restrict__ Ht,
                                 const float* __restrict__ a_l, const float* __restrict__ a_r, float* __restrict__ Al,
                                 float* __restrict__ Ar) {
  const bool vec = (f % 4) == 0;
  const int rpb = blockDim.x / h;  // rows per block step (h <= blockDim.x)
  const int rr = threadIdx.x / h, k = threadIdx.x - rr * h;
  if (rr >= rpb) return;
  const float* pl = a_l + k * f;
  const float* pr = a_r + k * f;
  const int64_t hf = (int64_t)h * f;
  for (int64_t v = (int64_t)blockIdx.x * rpb + rr; v < rows; v += (int64_t)gridDim.x * rpb) {
    const float* x = Ht + v * hf + (int64_t)k * f;
    float sl = 0.f, sr = 0.f;
    if (vec) {
      for (int j = 0; j < f; j += 4) {
        const float4 xv = __ldg(reinterpret_cast<const float4*>(x + j));
        const float4 lv = __ldg(reinterpret_cast<const float4*>(pl + j));
        const float4 rv = __ldg(reinterpret_cast<const float4*>(pr + j));
        sl = fmaf(xv.x, lv.x, sl); sl = fmaf(xv.y, lv.y, sl); sl = fmaf(xv.z, lv.z, sl); sl = fmaf(xv.w, lv.w, sl);
        sr = fmaf(xv.x, rv.x, sr); sr = fmaf(xv.y, rv.y, sr); sr = fmaf(xv.z, rv.z, sr); sr = fmaf(xv.w, rv.w, sr);
      }
    } else {
      for (int j = 0; j < f; ++j) {
        const float xv = __ldg(x + j);
        sl = fmaf(xv, __ldg(pl + j), sl);
        sr = fmaf(xv, __ldg(pr + j), sr);
      }
    }
    Al[v * h + k] = sl;
    Ar[v * h + k] = sr;
  }
}

constexpr int kGradBlocks = 1184;  // 8 per SM: enough independent row streams (C5: V = 10M)
// small tables (Cora: 2708 rows) take >= 32 rows per block instead of 2-3
inline int grad_blocks(int64_t rows) {
  const int64_t b = ceil_div(rows, (int64_t)32);
  return (int)(b < 1 ? 1 : b > kGradBlocks ? kGradBlocks : b);
}

// Per-block partial of da_l / da_r: threads = (row group, column quad) with 16-byte loads of
// Ht (hf % 4 == 0 and f % 4 == 0; else single columns); each thread walks its rows 4 at a time
// (independent loads in flight), then the row groups are combined in a fixed order ->
// deterministic.
__global__ void __launch_bounds__(256) attn_grad_partial_kernel(int64_t rows, int h, int f,
                                                                const float* __restrict__ Ht,
                                                                const float* __restrict__ dAl,
                                                                const float* __restrict__ dAr,
                                                                float* __restrict__ part) {
  __shared__ float red[2][256 * 4];
  const int hf = h * f;
  const int vw = (f % 4 == 0) ? 4 : 1;                          // columns per thread
  const int cw = min(hf - (int)blockIdx.y * 256 * vw, 256 * vw) / vw;  // column groups of this block
  const int RG = 256 / cw;                                      // row groups
  const int t = threadIdx.x, grp = t / cw, cl = t % cw;
  const int c = blockIdx.y * 256 * vw + cl * vw;                // first column of this thread
  const int k = c / f;
  const int64_t per = ceil_div(rows, (int64_t)gridDim.x);
  const int64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  float sl[4] = {0.f, 0.f, 0.f, 0.f}, sr[4] = {0.f, 0.f, 0.f, 0.f};
  if (grp < RG) {
    int64_t v = r0 + grp;
    if (vw == 4) {
      for (; v + 3 * RG < r1; v += 4 * RG) {
        float4 x[4];
        float l[4], r[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t vv = v + q * RG;
          x[q] = __ldg(reinterpret_cast<const float4*>(Ht + vv * hf + c));
          l[q] = __ldg(dAl + vv * h + k);
          r[q] = __ldg(dAr + vv * h + k);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          sl[0] = fmaf(l[q], x[q].x, sl[0]); sl[1] = fmaf(l[q], x[q].y, sl[1]);
          sl[2] = fmaf(l[q], x[q].z, sl[2]); sl[3] = fmaf(l[q], x[q].w, sl[3]);
          sr[0] = fmaf(r[q], x[q].x, sr[0]); sr[1] = fmaf(r[q], x[q].y, sr[1]);
          sr[2] = fmaf(r[q], x[q].z, sr[2]); sr[3] = fmaf(r[q], x[q].w, sr[3]);
        }
      }
      for (; v < r1; v += RG) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(Ht + v * hf + c));
        const float l = __ldg(dAl + v * h + k), r = __ldg(dAr + v * h + k);
        sl[0] = fmaf(l, x.x, sl[0]); sl[1] = fmaf(l, x.y, sl[1]); sl[2] = fmaf(l, x.z, sl[2]); sl[3] = fmaf(l, x.w, sl[3]);
        sr[0] = fmaf(r, x.x, sr[0]); sr[1] = fmaf(r, x.y, sr[1]); sr[2] = fmaf(r, x.z, sr[2]); sr[3] = fmaf(r, x.w, sr[3]);
      }
    } else {
      for (; v < r1; v += RG) {
        const float x = __ldg(Ht + v * hf + c);
        sl[0] = fmaf(__ldg(dAl + v * h + k), x, sl[0]);
        sr[0] = fmaf(__ldg(dAr + v * h + k), x, sr[0]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    red[0][t * 4 + q] = sl[q];
    red[1][t * 4 + q] = sr[q];
  }
  __syncthreads();
  if (grp == 0) {
    for (int g = 1; g < RG; ++g)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        sl[q] += red[0][(g * cw + cl) * 4 + q];
        sr[q] += red[1][(g * cw + cl) * 4 + q];
      }
    for (int q = 0; q < vw; ++q) {
      part[(int64_t)blockIdx.x * 2 * hf + c + q] = sl[q];
      part[(int64_t)blockIdx.x * 2 * hf + hf + c + q] = sr[q];
    }
  }
}

// Column c of the result = sum over blocks of the partials, one CTA per column (fixed order).
__global__ void __launch_bounds__(256) attn_grad_reduce_kernel(int nb, int hf, const float* __restrict__ part,
                                                               float* __restrict__ da_l, float* __restrict__ da_r) {
  __shared__ float sh[8];
  const int c = blockIdx.x;
  float s = 0.f;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) s += part[(int64_t)b * 2 * hf + c];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += sh[w];
    if (c < hf) da_l[c] = t; else da_r[c - hf] = t;
  }
}

// ---------------------------------------------------------------------------
// Dispatch over the compiled (VW, NV) variants.
// ---------------------------------------------------------------------------
enum class Kind { FwdOvl, BwdDst, BwdSrc, BwdSrcFast };
int num_sms();
bool pair_enabled();

template <int VW, int NV, int PER, int OCC>
void launch_fast_per(const GatParams& p, dim3 grid, cudaStream_t s) {
  if (p.ctr) gat_bwd_src_fast_kernel<VW, NV, PER, OCC, false, false, true><<<grid, THREADS, 0, s>>>(p);
  else gat_bwd_src_fast_kernel<VW, NV, PER, OCC><<<grid, THREADS, 0, s>>>(p);
}

template <int VW, int NV, int OCC>
void launch_fast(const GatParams& p, dim3 grid, cudaStream_t s) {
  constexpr int NVAL = GatherDepth<NV, OCC>::U * NV;
  grid.x = (unsigned)std::min<int64_t>(grid.x, (int64_t)num_sms() * (NV >= 8 ? 1 : OCC));  // persistent
  if (OCC == 2 && launch_bwd_src_lean(p, grid.x, s)) return;  // gat_lean.cu: the shapes that fill the warp
  if constexpr (NV == 2 && NVAL == 2 * 8) {
    // paired columns (8 lanes per head, two adjacent heads per lane, h = 8): the Reddit shape
    if (pair_enabled() && pair_lanes(p.h, p.f, VW, NV) == 8 && p.h == 8) {
      if (p.ctr) gat_bwd_src_fast_kernel<VW, NV, 8, OCC, false, true, true><<<grid, THREADS, 0, s>>>(p);
      else gat_bwd_src_fast_kernel<VW, NV, 8, OCC, false, true><<<grid, THREADS, 0, s>>>(p);
      return;
    }
  }
  switch (p.f / VW) {
    case 1: launch_fast_per<VW, NV, 1, OCC>(p, grid, s); break;
    case 2: if constexpr (NVAL % 2 == 0) launch_fast_per<VW, NV, 2, OCC>(p, grid, s); break;
    case 4: if constexpr (NVAL % 4 == 0) launch_fast_per<VW, NV, 4, OCC>(p, grid, s); break;
    case 8: if constexpr (NVAL % 8 == 0) launch_fast_per<VW, NV, 8, OCC>(p, grid, s); break;
    case 16: if constexpr (NVAL % 16 == 0) launch_fast_per<VW, NV, 16, OCC>(p, grid, s); break;
    default: break;  // excluded by gnncg_gat_fast_supported
  }
}

template <int VW, int NV, int OCC>
void launch_occ(Kind kind, const GatParams& p, dim3 grid, cudaStream_t s) {
  switch (kind) {
    case Kind::FwdOvl: {
      constexpr int U = GatherDepth<NV, OCC>::U;
      constexpr int MINB = NV >= 8 ? 1 : OCC;
      const unsigned g = (unsigned)std::min<int64_t>(grid.x, (int64_t)num_sms() * MINB);
      if (OCC == 2 && launch_fwd_lean(p, g, s)) break;  // gat_lean.cu: the shapes that fill the warp
      if (p.ctr) gat_fwd_ovl_kernel<VW, NV, U, WARPS, MINB, false, true><<<g, THREADS, 0, s>>>(p);
      else gat_fwd_ovl_kernel<VW, NV, U, WARPS, MINB><<<g, THREADS, 0, s>>>(p);
      break;
    }
    case Kind::BwdDst: gat_bwd_dst_kernel<VW, NV, OCC><<<grid, THREADS, 0, s>>>(p); break;
    case Kind::BwdSrc: gat_bwd_src_kernel<VW, NV, OCC><<<grid, THREADS, 0, s>>>(p); break;
    case Kind::BwdSrcFast: launch_fast<VW, NV, OCC>(p, grid, s); break;
  }
}

template <int VW, int NV>
void launch_variant(Kind kind, const GatParams& p, dim3 grid, cudaStream_t s) {
  launch_occ<VW, NV, 2>(kind, p, grid, s);  // 2 CTAs x 8 warps per SM (32 warps/SM measured slower)
}

template <int VW>
int launch_nv(Kind kind, const GatParams& p, dim3 grid, cudaStream_t s) {
  const int hf = p.h * p.f;
  const int nvec = (int)ceil_div(hf / VW, 32);
  if (nvec <= 1) launch_variant<VW, 1>(kind, p, grid, s);
  else if (nvec <= 2) launch_variant<VW, 2>(kind, p, grid, s);
  else if (nvec <= 4) launch_variant<VW, 4>(kind, p, grid, s);
  else if (nvec <= 8) launch_variant<VW, 8>(kind, p, grid, s);
  else return fail(GNNCG_ERR_UNSUPPORTED, "gat: h*f = %d exceeds the compiled limit %d", hf, 256 * VW);
  return GNNCG_OK;
}

int dispatch(Kind kind, const GatParams& p, cudaStream_t s) {
  if (p.num_items == 0) return GNNCG_OK;
  dim3 grid((unsigned)ceil_div(p.num_items, WARPS));
  int rc;
  if (p.f % 4 == 0) rc = launch_nv<4>(kind, p, grid, s);
  else if (p.f % 2 == 0) rc = launch_nv<2>(kind, p, grid, s);
  else rc = launch_nv<1>(kind, p, grid, s);
  if (rc != GNNCG_OK) return rc;
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

// bf16 gather table: lane width VW = 8 when the row fills whole 256-column warps, else 4.
int lp_width(int h, int f) {
  const int hf = h * f;
  if (h < 1 || h > MAXH) return 0;
  if (f % 8 == 0 && hf % 256 == 0 && hf <= 512) return 8;
  if (f % 4 == 0 && hf <= 256) return 4;
  return 0;
}

template <int VW, int NV>
bool lp_fast_ok(int f) {
  constexpr int NVAL = LpDepth<VW, NV>::U * NV;
  const int per = f / VW;
  return per >= 1 && per <= 16 && (per & (per - 1)) == 0 && NVAL % per == 0;
}

template <int VW, int NV, int PER>
void launch_lp_fast_per(const GatParams& p, unsigned g, cudaStream_t s) {
  constexpr int NVAL = LpDepth<VW, NV>::U * NV;
  if constexpr (NVAL % PER == 0) {
    if (p.ctr) gat_bwd_src_fast_kernel<VW, NV, PER, 2, true, false, true><<<g, THREADS, 0, s>>>(p);
    else gat_bwd_src_fast_kernel<VW, NV, PER, 2, true><<<g, THREADS, 0, s>>>(p);
  }
}

template <int VW, int NV>
void launch_lp(Kind kind, const GatParams& p, cudaStream_t s) {
  const unsigned g = (unsigned)std::min<int64_t>(ceil_div(p.num_items, WARPS), (int64_t)num_sms() * 2);
  // gat_lean.cu: the 8 x 32 / 8 x 16 shapes
  if (kind == Kind::FwdOvl && launch_fwd_lean_lp(p, s)) return;
  if (kind == Kind::BwdSrcFast && launch_bwd_src_lean_lp(p, s)) return;
  if (kind == Kind::FwdOvl) {
    if (p.ctr) gat_fwd_ovl_kernel<VW, NV, LpDepth<VW, NV>::U, WARPS, 2, true, true><<<g, THREADS, 0, s>>>(p);
    else gat_fwd_ovl_kernel<VW, NV, LpDepth<VW, NV>::U, WARPS, 2, true><<<g, THREADS, 0, s>>>(p);
  } else {
    switch (p.f / VW) {
      case 1: launch_lp_fast_per<VW, NV, 1>(p, g, s); break;
      case 2: launch_lp_fast_per<VW, NV, 2>(p, g, s); break;
      case 4: launch_lp_fast_per<VW, NV, 4>(p, g, s); break;
      case 8: launch_lp_fast_per<VW, NV, 8>(p, g, s); break;
      case 16: launch_lp_fast_per<VW, NV, 16>(p, g, s); break;
      default: break;  // excluded by gnncg_gat_bf16_supported
    }
  }
}

int dispatch_lp(Kind kind, const GatParams& p, cudaStream_t s) {
  if (p.num_items == 0) return GNNCG_OK;
  const int hf = p.h * p.f, vw = lp_width(p.h, p.f);
  if (vw == 8) {
    if (hf <= 256) launch_lp<8, 1>(kind, p, s);
    else launch_lp<8, 2>(kind, p, s);
  } else if (vw == 4) {
    if (hf <= 128) launch_lp<4, 1>(kind, p, s);
    else launch_lp<4, 2>(kind, p, s);
  } else {
    return fail(GNNCG_ERR_UNSUPPORTED, "gat bf16 gather: heads=%d f=%d unsupported", p.h, p.f);
  }
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

// fp32 -> bf16, round to nearest even (the gather tables of the bf16 mode).
__global__ void pack_bf16_kernel(int64_t n, const float* __restrict__ src, uint16_t* __restrict__ dst) {
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(src) + i);
    const uint32_t lo = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v.x)) |
                        ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v.y)) << 16);
    const uint32_t hi = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v.z)) |
                        ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v.w)) << 16);
    reinterpret_cast<uint2*>(dst)[i] = make_uint2(lo, hi);
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __bfloat16_as_ushort(__float2bfloat16_rn(src[i]));
}

}  // namespace


namespace {


// K2 / K4f pull work items from a counter in the workspace (behind the partials, where
// gnncg_gat_workspace reserves 256 bytes) instead of a fixed stride: the items are ordered
// largest first, so warps take them longest-first and finish together (with a fixed stride
// the busiest warp carries ~11% more edges than the mean on the Reddit shape, simulated).  Measured: K2 7.94 ->
// 7.47 ms, K4f 11.75 -> 11.1 ms; C5 K4f 132.5 -> 115.8 ms with 5 items per request.
// GNNCG_GAT_DYN=0 restores the fixed stride; a workspace without the counter bytes also does.
// GNNCG_GAT_DYN_BATCH caps the items per counter request (default 8; 1 = one at a time)
uint64_t dyn_batch_cap() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("GNNCG_GAT_DYN_BATCH");
    v = e ? std::max(1, atoi(e)) : 8;
  }
  return (uint64_t)v;
}

// 0: fixed stride; 1: counter for graphs with >= 8 items per warp (default); 2: counter always
// (tests: it exercises the counter and K4f's batched requests on small graphs)
int dyn_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("GNNCG_GAT_DYN");
    v = e ? atoi(e) : 1;
  }
  return v;
}
bool dyn_enabled() { return dyn_mode() >= 1; }

int attach_counter(GatParams& p, uint64_t num_edges, void* ws, size_t ws_bytes, size_t need, cudaStream_t s) {
  p.ctr = nullptr;
  // no items (a rank whose block has no in-edges): nothing to fetch, and no mean to take
  if (p.num_items <= 0 || !dyn_enabled() || !ws || ws_bytes < align_up(need) + sizeof(unsigned)) return GNNCG_OK;
  // a few items per warp of the persistent grid balance themselves (Cora: 2708 items; the
  // counter's memset cost more than it saved there)
  const uint64_t warps = (uint64_t)num_sms() * 2 * WARPS;
  if (dyn_mode() == 1 && (uint64_t)p.num_items < 8 * warps) return GNNCG_OK;
  // K4f: about 512 edges per request (Reddit, 452 edges per item: 1; C5: 5)
  const uint64_t mean = num_edges / (uint64_t)p.num_items;
  p.batch = (int)std::max<uint64_t>(1, std::min<uint64_t>(dyn_batch_cap(), 512 / std::max<uint64_t>(mean, 1)));
  // the counter is 32-bit and every warp makes one request past the end: keep it from
  // wrapping (schedule item ids are u32, so this only bites near 2^32 items)
  if ((uint64_t)p.num_items + warps * (uint64_t)p.batch >= (1ull << 32)) return GNNCG_OK;
  p.ctr = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + align_up(need));
  GNNCG_CUDA_TRY(cudaMemsetAsync(p.ctr, 0, sizeof(unsigned), s));
  return GNNCG_OK;
}


// GNNCG_GAT_PAIR=0 disables K4f's paired-head column mapping.
bool pair_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("GNNCG_GAT_PAIR");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int num_sms() {
  static int v = 0;
  if (v == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
  }
  return v;
}

int check_common(const gnncg_index_t* idx, const gnncg_sched_t* sched, int h, int f) {
  GNNCG_REQUIRE(idx && sched, GNNCG_ERR_ARG, "gat: null index or schedule");
  GNNCG_REQUIRE(h >= 1 && h <= MAXH, GNNCG_ERR_UNSUPPORTED, "gat: heads=%d outside [1,%d]", h, MAXH);
  GNNCG_REQUIRE(f >= 1, GNNCG_ERR_SHAPE, "gat: f must be >= 1");
  GNNCG_REQUIRE(idx->num_rows >= 0 && (idx->num_rows == 0 || idx->off), GNNCG_ERR_ARG, "gat: bad index");
  GNNCG_REQUIRE(sched->num_items == 0 || sched->items, GNNCG_ERR_ARG, "gat: bad schedule");
  GNNCG_REQUIRE(sched->chunk >= 32, GNNCG_ERR_ARG, "gat: schedule chunk < 32");
  return GNNCG_OK;
}

size_t fwd_part_bytes(const gnncg_sched_t* s, int h, int f) {
  return s ? (size_t)s->num_split_items * (size_t)fwd_stride(h, f) * sizeof(float) : 0;
}
size_t dst_part_bytes(const gnncg_sched_t* s, int h) {
  return s ? (size_t)s->num_split_items * (size_t)(3 * h) * sizeof(float) : 0;
}
size_t src_part_bytes(const gnncg_sched_t* s, int h, int f) {
  return s ? (size_t)s->num_split_items * (size_t)src_stride(h, f) * sizeof(float) : 0;
}

}  // namespace
}  // namespace gnncg_b200

using namespace gnncg_b200;

extern "C" {

int gnncg_gat_attn_dots(int64_t rows, int h, int f, const float* Ht, const float* a_l, const float* a_r, float* Al,
                        float* Ar, void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(rows >= 0 && h >= 1 && f >= 1, GNNCG_ERR_SHAPE, "attn_dots: bad shape");
  if (rows == 0) return GNNCG_OK;
  GNNCG_REQUIRE(Ht && a_l && a_r && Al && Ar, GNNCG_ERR_ARG, "attn_dots: null pointer");
  GNNCG_REQUIRE(h <= 256, GNNCG_ERR_UNSUPPORTED, "attn_dots: heads=%d > 256", h);
  const int rpb = 256 / h;
  const int g = (int)std::min<int64_t>(ceil_div(rows, (int64_t)rpb), 148 * 32);
  cost_add(kCostLp, (uint64_t)rows, 1, as_stream(stream));
  attn_dots_kernel<<<g, 256, 0, as_stream(stream)>>>(rows, h, f, Ht, a_l, a_r, Al, Ar);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

size_t gnncg_gat_workspace(const gnncg_sched_t* dst_sched, const gnncg_sched_t* src_sched, int h, int f) {
  size_t b = fwd_part_bytes(dst_sched, h, f);
  b = std::max(b, dst_part_bytes(dst_sched, h));
  b = std::max(b, src_part_bytes(src_sched, h, f));
  return align_up(b) + 256;  // + the work counter of the persistent TMA-fed kernels
}

static int gat_fwd_impl(bool lp, const gnncg_index_t* csr_dst, const gnncg_sched_t* sched, int h, int f, float slope,
                        const float* Ht, const uint16_t* Ht_lp, const float* Al, const float* Ar, float* out, float* m,
                        float* d, void* ws, size_t ws_bytes, void* stream) {
  GNNCG_DEVICE_GUARD();
  int rc = check_common(csr_dst, sched, h, f);
  if (rc) return rc;
  if (sched->num_items == 0) return GNNCG_OK;
  GNNCG_REQUIRE((lp ? Ht_lp != nullptr : Ht != nullptr) && Al && Ar && out && m && d &&
                    (csr_dst->num_edges == 0 || csr_dst->nbr),
                GNNCG_ERR_ARG, "gat_fwd: null pointer");
  const size_t need = fwd_part_bytes(sched, h, f);
  GNNCG_REQUIRE(ws_bytes >= need && (need == 0 || ws), GNNCG_ERR_WORKSPACE, "gat_fwd: workspace %zu < %zu",
                ws_bytes, need);
  GatParams p{};
  p.cnt = cost_slot(kCostK2);
  p.off = csr_dst->off; p.nbr = csr_dst->nbr; p.items = sched->items;
  p.num_items = sched->num_items; p.num_split_items = sched->num_split_items; p.chunk = sched->chunk;
  p.h = h; p.f = f; p.slope = slope;
  p.Ht = Ht; p.lp = Ht_lp; p.Al = Al; p.Ar = Ar; p.out = out; p.mo = m; p.dd = d; p.part = static_cast<float*>(ws);
  if (!lp) p.win = l2_window(sched, Ht, (size_t)h * f * 4);  // source rows of Ht (csc_src offsets)
  cudaStream_t s = as_stream(stream);
  if (lp) {
    rc = attach_counter(p, csr_dst->num_edges, ws, ws_bytes, need, s);
    if (rc) return rc;
    rc = dispatch_lp(Kind::FwdOvl, p, s);
  } else {
    rc = attach_counter(p, csr_dst->num_edges, ws, ws_bytes, need, s);
    if (rc) return rc;
    rc = dispatch(Kind::FwdOvl, p, s);
  }
  if (rc) return rc;
  if (sched->num_split_rows > 0) {
    gat_fwd_merge_kernel<<<(unsigned)ceil_div(sched->num_split_rows, WARPS), THREADS, 0, s>>>(
        p, sched->split_rows, sched->split_first, sched->num_split_rows);
    GNNCG_LAUNCH_CHECK();
  }
  return GNNCG_OK;
}

int gnncg_gat_fwd(const gnncg_index_t* csr_dst, const gnncg_sched_t* sched, int h, int f, float slope,
                  const float* Ht, const float* Al, const float* Ar, float* out, float* m, float* d, void* ws,
                  size_t ws_bytes, void* stream) {
  return gat_fwd_impl(false, csr_dst, sched, h, f, slope, Ht, nullptr, Al, Ar, out, m, d, ws, ws_bytes, stream);
}

int gnncg_gat_bf16_supported(int h, int f) {
  const int vw = lp_width(h, f);
  if (vw == 8) return h * f <= 256 ? lp_fast_ok<8, 1>(f) : lp_fast_ok<8, 2>(f);
  if (vw == 4) return h * f <= 128 ? lp_fast_ok<4, 1>(f) : lp_fast_ok<4, 2>(f);
  return 0;
}

int gnncg_pack_bf16(int64_t n, const float* src, uint16_t* dst, void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(n >= 0, GNNCG_ERR_SHAPE, "pack_bf16: n < 0");
  if (n == 0) return GNNCG_OK;
  GNNCG_REQUIRE(src && dst, GNNCG_ERR_ARG, "pack_bf16: null pointer");
  GNNCG_REQUIRE(((uintptr_t)src & 15) == 0 && ((uintptr_t)dst & 7) == 0, GNNCG_ERR_ARG, "pack_bf16: misaligned");
  const int g = (int)std::min<int64_t>(ceil_div(n / 4 + 1, 256), 148 * 16);
  pack_bf16_kernel<<<g, 256, 0, as_stream(stream)>>>(n, src, dst);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

int gnncg_gat_fwd_bf16(const gnncg_index_t* csr_dst, const gnncg_sched_t* sched, int h, int f, float slope,
                       const uint16_t* Ht_bf16, const float* Al, const float* Ar, float* out, float* m, float* d,
                       void* ws, size_t ws_bytes, void* stream) {
  GNNCG_REQUIRE(gnncg_gat_bf16_supported(h, f), GNNCG_ERR_UNSUPPORTED, "gat_fwd_bf16: heads=%d f=%d unsupported",
                h, f);
  return gat_fwd_impl(true, csr_dst, sched, h, f, slope, nullptr, Ht_bf16, Al, Ar, out, m, d, ws, ws_bytes, stream);
}

int gnncg_gat_bwd_dst(const gnncg_index_t* csr_dst, const gnncg_sched_t* sched, int h, int f, float slope,
                      const float* Ht, const float* Al, const float* Ar, const float* m, const float* d,
                      const float* dOut, float* c, float* dAr, void* ws, size_t ws_bytes, void* stream) {
  GNNCG_DEVICE_GUARD();
  int rc = check_common(csr_dst, sched, h, f);
  if (rc) return rc;
  if (sched->num_items == 0) return GNNCG_OK;
  GNNCG_REQUIRE(Ht && Al && Ar && m && d && dOut && c && dAr && (csr_dst->num_edges == 0 || csr_dst->nbr), GNNCG_ERR_ARG,
                "gat_bwd_dst: null pointer");
  const size_t need = dst_part_bytes(sched, h);
  GNNCG_REQUIRE(ws_bytes >= need && (need == 0 || ws), GNNCG_ERR_WORKSPACE, "gat_bwd_dst: workspace %zu < %zu",
                ws_bytes, need);
  GatParams p{};
  p.cnt = cost_slot(kCostK3);
  p.off = csr_dst->off; p.nbr = csr_dst->nbr; p.items = sched->items;
  p.num_items = sched->num_items; p.num_split_items = sched->num_split_items; p.chunk = sched->chunk;
  p.h = h; p.f = f; p.slope = slope;
  p.Ht = Ht; p.Al = Al; p.Ar = Ar; p.m = m; p.d = d; p.dOut = dOut; p.co = c; p.dAro = dAr;
  p.part = static_cast<float*>(ws);
  cudaStream_t s = as_stream(stream);
  rc = dispatch(Kind::BwdDst, p, s);
  if (rc) return rc;
  if (sched->num_split_rows > 0) {
    const int64_t n = sched->num_split_rows * h;
    gat_bwd_dst_merge_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(p, sched->split_rows, sched->split_first,
                                                                        sched->num_split_rows);
    GNNCG_LAUNCH_CHECK();
  }
  return GNNCG_OK;
}

int gnncg_gat_bwd_src(const gnncg_index_t* csc_src, const gnncg_sched_t* sched, int h, int f, float slope,
                      int64_t row_base, int64_t num_local, const float* Ht, const float* Al, const float* Ar,
                      const float* m, const float* d, const float* c, const float* dOut, const float* dAr,
                      const float* a_l, const float* a_r, float* dHt, float* dAl, void* ws, size_t ws_bytes,
                      void* stream) {
  GNNCG_DEVICE_GUARD();
  int rc = check_common(csc_src, sched, h, f);
  if (rc) return rc;
  if (sched->num_items == 0) return GNNCG_OK;
  GNNCG_REQUIRE(Ht && Al && Ar && m && d && c && dOut && dAr && a_l && a_r && dHt && dAl, GNNCG_ERR_ARG,
                "gat_bwd_src: null pointer");
  GNNCG_REQUIRE(row_base >= 0 && num_local >= 0, GNNCG_ERR_ARG, "gat_bwd_src: bad row block");
  const size_t need = src_part_bytes(sched, h, f);
  GNNCG_REQUIRE(ws_bytes >= need && (need == 0 || ws), GNNCG_ERR_WORKSPACE, "gat_bwd_src: workspace %zu < %zu",
                ws_bytes, need);
  GatParams p{};
  p.cnt = cost_slot(kCostK4);
  p.off = csc_src->off; p.nbr = csc_src->nbr; p.items = sched->items;
  p.num_items = sched->num_items; p.num_split_items = sched->num_split_items; p.chunk = sched->chunk;
  p.h = h; p.f = f; p.slope = slope;
  p.Ht = Ht; p.Al = Al; p.Ar = Ar; p.m = m; p.d = d; p.c = c; p.dOut = dOut; p.dAr = dAr;
  p.a_l = a_l; p.a_r = a_r; p.dHt = dHt; p.dAl = dAl; p.row_base = row_base; p.num_local = num_local;
  p.part = static_cast<float*>(ws);
  cudaStream_t s = as_stream(stream);
  rc = dispatch(Kind::BwdSrc, p, s);
  if (rc) return rc;
  if (sched->num_split_rows > 0) {
    gat_bwd_src_merge_kernel<<<(unsigned)ceil_div(sched->num_split_rows, WARPS), THREADS, 0, s>>>(
        p, sched->split_rows, sched->split_first, sched->num_split_rows);
    GNNCG_LAUNCH_CHECK();
  }
  return GNNCG_OK;
}

int gnncg_gat_fast_supported(int h, int f) {
  const int vw = f % 4 == 0 ? 4 : (f % 2 == 0 ? 2 : 1);
  const int per = f / vw;
  if (h < 1 || h > MAXH || per < 1 || per > 16 || (per & (per - 1)) != 0 || h * f > 256 * vw) return 0;
  const int nvec = (int)ceil_div(h * f / vw, 32);
  const int nv = nvec <= 1 ? 1 : nvec <= 2 ? 2 : nvec <= 4 ? 4 : 8;
  const int u = nv <= 2 ? 8 : (nv == 4 ? 4 : 2);
  return (u * nv) % per == 0;
}

int gnncg_gat_rec_stride(int h) { return rec_stride(h); }

int gnncg_gat_bwd_prep(int64_t rows, int h, int f, const float* dOut, const float* out, const float* Ar,
                       const float* m, const float* d, float* rec, void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(rows >= 0 && h >= 1 && h <= MAXH && f >= 1, GNNCG_ERR_SHAPE, "gat_bwd_prep: bad shape");
  if (rows == 0) return GNNCG_OK;
  GNNCG_REQUIRE(dOut && out && Ar && m && d && rec, GNNCG_ERR_ARG, "gat_bwd_prep: null pointer");
  const int g = (int)std::min<int64_t>(ceil_div(rows * h, 256), 148 * 32);
  gat_bwd_prep_kernel<<<g, 256, 0, as_stream(stream)>>>(rows, h, f, dOut, out, Ar, m, d, rec);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

static int gat_bwd_src_fused_impl(bool lp, const gnncg_index_t* csc_src, const gnncg_sched_t* sched, int h, int f,
                                  float slope, int64_t row_base, int64_t num_local, const float* Ht,
                                  const uint16_t* Ht_lp, const float* Al,
                                  const float* dst_rec, const float* dOut, const uint16_t* dOut_lp, const float* a_l,
                                  const float* a_r, float* dHt, float* dAl, float* dAr, void* ws, size_t ws_bytes,
                                  void* stream, int flags = 0) {
  GNNCG_DEVICE_GUARD();
  int rc = check_common(csc_src, sched, h, f);
  if (rc) return rc;
  if (lp) {
    GNNCG_REQUIRE(gnncg_gat_bf16_supported(h, f), GNNCG_ERR_UNSUPPORTED,
                  "gat_bwd_src_fused_bf16: heads=%d f=%d unsupported", h, f);
  } else {
    GNNCG_REQUIRE(gnncg_gat_fast_supported(h, f), GNNCG_ERR_UNSUPPORTED,
                  "gat_bwd_src_fused: f/VW must be a power of two <= 32 (use gnncg_gat_bwd_dst + gnncg_gat_bwd_src)");
  }
  if (sched->num_items == 0 && num_local == 0) return GNNCG_OK;  // empty graph
  GNNCG_REQUIRE((lp ? (Ht_lp && dOut_lp) : (Ht && dOut)) && Al && dst_rec && a_l && a_r && dHt && dAl && dAr,
                GNNCG_ERR_ARG, "gat_bwd_src_fused: null pointer");
  GNNCG_REQUIRE(row_base >= 0 && num_local >= 0, GNNCG_ERR_ARG, "gat_bwd_src_fused: bad row block");
  const size_t need = src_part_bytes(sched, h, f);
  GNNCG_REQUIRE(ws_bytes >= need && (need == 0 || ws), GNNCG_ERR_WORKSPACE,
                "gat_bwd_src_fused: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = as_stream(stream);
  if (!(flags & kFusedKeepDar)) GNNCG_CUDA_TRY(cudaMemsetAsync(dAr, 0, sizeof(float) * (size_t)num_local * h, s));
  GatParams p{};
  p.cnt = cost_slot(kCostK4f);
  p.off = csc_src->off; p.nbr = csc_src->nbr; p.items = sched->items;
  p.num_items = sched->num_items; p.num_split_items = sched->num_split_items; p.chunk = sched->chunk;
  p.h = h; p.f = f; p.slope = slope;
  p.Ht = Ht; p.Al = Al; p.rec = dst_rec; p.dOut = dOut; p.lp = dOut_lp; p.lp_x = Ht_lp; p.dAr = dAr; p.dAro = dAr;
  p.a_l = a_l; p.a_r = a_r; p.dHt = dHt; p.dAl = dAl; p.row_base = row_base; p.num_local = num_local;
  p.part = static_cast<float*>(ws);
  p.fast = 1;
  if (!lp) p.win = l2_window(sched, dOut, (size_t)h * f * 4);  // destination rows of dOut (csr_dst offsets)
  // (C5's ~100-edge items: one item per request was slower than the fixed stride, 132.5 ->
  // 134.6 ms, the counter address being the limit; 5 per request: 115.8 ms)
  rc = attach_counter(p, csc_src->num_edges, ws, ws_bytes, need, s);
  if (rc) return rc;
  rc = lp ? dispatch_lp(Kind::BwdSrcFast, p, s) : dispatch(Kind::BwdSrcFast, p, s);
  if (rc) return rc;
  if (sched->num_split_rows > 0) {
    gat_bwd_src_merge_kernel<<<(unsigned)ceil_div(sched->num_split_rows, WARPS), THREADS, 0, s>>>(
        p, sched->split_rows, sched->split_first, sched->num_split_rows);
    GNNCG_LAUNCH_CHECK();
  }
  if (num_local > 0 && !(flags & kFusedNoLpDar)) {
    const int g = (int)std::min<int64_t>(ceil_div(num_local * h * f, 256), 148 * 32);
    const int threads = (f % 4 == 0 && h * f / 4 <= 1024) ? std::max(256, h * f / 4) : 256;
    gat_lp_dar_kernel<<<g, threads, 0, s>>>(num_local, row_base, h, f, dAr, a_r, dHt);
    GNNCG_LAUNCH_CHECK();
  }
  return GNNCG_OK;
}


int gnncg_gat_bwd_prep_bf16(int64_t rows, int h, int f, const float* dOut, const float* out, const float* Ar,
                            const float* m, const float* d, float* rec, uint16_t* dOut_bf16, void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(rows >= 0 && h >= 1 && h <= MAXH && f >= 4 && f % 4 == 0, GNNCG_ERR_SHAPE,
                "gat_bwd_prep_bf16: bad shape");
  if (rows == 0) return GNNCG_OK;
  GNNCG_REQUIRE(dOut && out && Ar && m && d && rec && dOut_bf16, GNNCG_ERR_ARG, "gat_bwd_prep_bf16: null pointer");
  const int g = (int)std::min<int64_t>(ceil_div(rows * h, 256), 148 * 32);
  gat_bwd_prep_bf16_kernel<<<g, 256, 0, as_stream(stream)>>>(rows, h, f, dOut, out, Ar, m, d, rec, dOut_bf16);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

int gnncg_gat_bwd_src_fused(const gnncg_index_t* csc_src, const gnncg_sched_t* sched, int h, int f, float slope,
                            int64_t row_base, int64_t num_local, const float* Ht, const float* Al,
                            const float* dst_rec, const float* dOut, const float* a_l, const float* a_r, float* dHt,
                            float* dAl, float* dAr, void* ws, size_t ws_bytes, void* stream) {
  return gat_bwd_src_fused_impl(false, csc_src, sched, h, f, slope, row_base, num_local, Ht, nullptr, Al, dst_rec, dOut,
                                nullptr, a_l, a_r, dHt, dAl, dAr, ws, ws_bytes, stream);
}

int gnncg_gat_bwd_src_fused_bf16(const gnncg_index_t* csc_src, const gnncg_sched_t* sched, int h, int f,
                                 float slope, int64_t row_base, int64_t num_local, const uint16_t* Ht_bf16,
                                 const float* Al, const float* dst_rec, const uint16_t* dOut_bf16, const float* a_l,
                                 const float* a_r, float* dHt, float* dAl, float* dAr, void* ws, size_t ws_bytes,
                                 void* stream) {
  return gat_bwd_src_fused_impl(true, csc_src, sched, h, f, slope, row_base, num_local, nullptr, Ht_bf16, Al, dst_rec,
                                nullptr, dOut_bf16, a_l, a_r, dHt, dAl, dAr, ws, ws_bytes, stream);
}

size_t gnncg_gat_attn_grad_workspace(int64_t rows, int h, int f) {
  return align_up((size_t)grad_blocks(rows) * 2 * h * f * sizeof(float));
}

int gnncg_gat_attn_grad(int64_t rows, int h, int f, const float* Ht, const float* dAl, const float* dAr,
                        float* da_l, float* da_r, void* ws, size_t ws_bytes, void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(rows >= 0 && h >= 1 && f >= 1, GNNCG_ERR_SHAPE, "attn_grad: bad shape");
  GNNCG_REQUIRE(da_l && da_r && (rows == 0 || (Ht && dAl && dAr)), GNNCG_ERR_ARG, "attn_grad: null pointer");
  const size_t need = gnncg_gat_attn_grad_workspace(rows, h, f);
  GNNCG_REQUIRE(ws_bytes >= need && ws, GNNCG_ERR_WORKSPACE, "attn_grad: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = as_stream(stream);
  const int hf = h * f;
  float* part = static_cast<float*>(ws);
  const int nb = grad_blocks(rows);
  dim3 g1(nb, (unsigned)ceil_div(hf, f % 4 == 0 ? 1024 : 256));
  attn_grad_partial_kernel<<<g1, 256, 0, s>>>(rows, h, f, Ht, dAl, dAr, part);
  GNNCG_LAUNCH_CHECK();
  attn_grad_reduce_kernel<<<(unsigned)(2 * hf), 256, 0, s>>>(nb, hf, part, da_l, da_r);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

}  // extern "C"

namespace gnncg_b200 {

// One K4f pass of the partitioned backward (csrc/dist.cu): fp32 tables, dA_r zeroed only
// when asked, the dA_r (x) a_r LP term left to the caller (it needs every pass's reductions).
int gat_bwd_src_fused_pass(const gnncg_index_t* csc_src, const gnncg_sched_t* sched, int h, int f, float slope,
                           int64_t num_local, const float* Ht, const float* Al, const float* dst_rec,
                           const float* dOut, const float* a_l, const float* a_r, float* dHt, float* dAl, float* dAr,
                           bool zero_dar, void* ws, size_t ws_bytes, cudaStream_t stream) {
  return gat_bwd_src_fused_impl(false, csc_src, sched, h, f, slope, 0, num_local, Ht, nullptr, Al, dst_rec, dOut,
                                nullptr, a_l, a_r, dHt, dAl, dAr, ws, ws_bytes, stream,
                                kFusedNoLpDar | (zero_dar ? 0 : kFusedKeepDar));
}

// dHt[r, :] += dA_r[r] (x) a_r over rows [0, rows) (the fast-mode LP epilogue, dist.cu).
int gat_lp_dar(int64_t rows, int h, int f, const float* dAr, const float* a_r, float* dHt, cudaStream_t s) {
  if (rows <= 0) return GNNCG_OK;
  const int g = (int)std::min<int64_t>(ceil_div(rows * h * f, 256), 148 * 32);
  const int threads = (f % 4 == 0 && h * f / 4 <= 1024) ? std::max(256, h * f / 4) : 256;
  gat_lp_dar_kernel<<<g, threads, 0, s>>>(rows, 0, h, f, dAr, a_r, dHt);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

}  // namespace gnncg_b200
