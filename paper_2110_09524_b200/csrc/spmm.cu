// SPDX-License-Identifier: Apache-2.0
//
// Weighted Aggregate (GCN): the spec's GCN layer
//   build_model(gcn) = [ApplyVertex(W), Scatter(copy_u), ApplyEdge(x e_uv), Gather(sum),
//                       ApplyVertex(+b, sigma)]
// with the graph part fused into one kernel over an index:
//   Y[r, :] = act( b + sum_{i in row r} w[eid_i] * X[nbr_i, :] )
// Forward: index = csr_dst, X = H W.  Backward: index = csc_src, X = dZ (= dOut masked by the
// ReLU of the forward output), no bias/activation -- the transpose of the same aggregate.
// Same unified thread mapping as the GAT kernels (gat.cu): one warp per work item (and column
// slice), the 32-edge block's ids and weights held one per lane and broadcast by shuffle,
// 16-byte column gathers, hub rows split with fixed-order partial merges (deterministic).
#include "common.cuh"
#include "gat_common.cuh"

#include <algorithm>
#include <cstdint>
#include <cstdlib>

namespace gnncg_b200 {
namespace {

using namespace gat;

struct SpmmParams {
  const uint64_t* off;
  const uint32_t* nbr;
  const uint32_t* eid;
  const uint32_t* items;
  int64_t num_items, num_split_items;
  int chunk, cols, tile;  // tile = columns per blockIdx.y slice (multiple of VW)
  const float *w, *X, *bias;
  float *Y, *part;
  int relu;
};

// Rows gathered per step (U) for a given per-lane width NV and CTAs/SM OCC: the register
// budget (255 / 128 / 64 / 32 for OCC 1 / 2 / 4 / 8) bounds U * NV float4s in flight.
template <int NV, int OCC>
struct SpmmDepth {
  static constexpr int U = OCC >= 8 ? (NV == 1 ? 4 : (NV == 2 ? 2 : 1))
                                    : GatherDepth<NV, OCC>::U;
};

template <int VW, int NV, int OCC>
__global__ void __launch_bounds__(THREADS, OCC) spmm_kernel(SpmmParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t wi = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (wi >= p.num_items) return;
  const Item it = decode_item(p.items, p.off, wi, p.num_split_items, p.chunk);
  const int F = p.cols;
  // column slice of this CTA row (wide feature matrices are split over blockIdx.y)
  const int c0 = blockIdx.y * p.tile, c1 = min(F, c0 + p.tile);
  Cols<VW, NV> cols(lane, F, F);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    cols.col[i] += c0;
    cols.ok[i] = cols.col[i] < c1;
  }
  Vec<VW> acc[NV];
  zero(acc);
  constexpr int U = SpmmDepth<NV, OCC>::U;
  // Lane j holds edge j of the current 32-edge block (neighbour id, weight) in registers and
  // the warp reads them by shuffle.  The next block's ids are loaded before the current
  // block's gathers; its weights (a dependent load through eid) after them.
  uint32_t nb = 0;
  float a = 0.f;
  if (it.e0 + lane < it.e1) {
    nb = __ldg(p.nbr + it.e0 + lane);
    a = p.w ? __ldg(p.w + __ldg(p.eid + it.e0 + lane)) : 1.f;
  }
  for (uint64_t base = it.e0; base < it.e1; base += 32) {
    const int n = (int)min((uint64_t)32, it.e1 - base);
    const uint64_t nx = base + 32 + lane;
    const bool has_next = nx < it.e1;
    uint32_t nb_n = 0, eid_n = 0;
    if (has_next) {
      nb_n = __ldg(p.nbr + nx);
      if (p.w) eid_n = __ldg(p.eid + nx);
    }
    int j = 0;
    for (; j + U <= n; j += U) {
      Vec<VW> x[U][NV];
#pragma unroll
      for (int t = 0; t < U; ++t) gather_row<VW, NV>(p.X, __shfl_sync(0xffffffffu, nb, j + t), F, cols, x[t]);
#pragma unroll
      for (int t = 0; t < U; ++t) {
        const float at = __shfl_sync(0xffffffffu, a, j + t);
#pragma unroll
        for (int i = 0; i < NV; ++i)
#pragma unroll
          for (int q = 0; q < VW; ++q) acc[i].x[q] = fmaf(at, x[t][i].x[q], acc[i].x[q]);
      }
    }
    for (; j < n; ++j) {
      Vec<VW> x[NV];
      gather_row<VW, NV>(p.X, __shfl_sync(0xffffffffu, nb, j), F, cols, x);
      const float at = __shfl_sync(0xffffffffu, a, j);
#pragma unroll
      for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int q = 0; q < VW; ++q) acc[i].x[q] = fmaf(at, x[i].x[q], acc[i].x[q]);
    }
    nb = nb_n;
    a = has_next ? (p.w ? __ldg(p.w + eid_n) : 1.f) : 0.f;
  }
  if (!it.split) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      if (cols.ok[i]) {
        Vec<VW> o;
#pragma unroll
        for (int q = 0; q < VW; ++q) {
          float z = acc[i].x[q] + (p.bias ? __ldg(p.bias + cols.col[i] + q) : 0.f);
          o.x[q] = p.relu ? fmaxf(z, 0.f) : z;
        }
        st_vec<VW>(p.Y + (int64_t)it.row * F + cols.col[i], o);
      }
    }
  } else {
    float* part = p.part + wi * (int64_t)F;
#pragma unroll
    for (int i = 0; i < NV; ++i)
      if (cols.ok[i]) st_vec<VW>(part + cols.col[i], acc[i]);
  }
}

// Lean weighted aggregate for 256-column rows (the GCN hidden width; K2's layout without the
// softmax): each lane owns 8 consecutive columns and gathers them with one 256-bit load; the
// block's ids and weights sit in shared memory (one broadcast LDS.128 per 4 rows instead of two
// shuffles per row); 8 rows in flight per warp; ids read evict-first; the next block's weight
// (a dependent load through eid) goes out after the first row group's gathers.
struct SpmmLeanSmem {
  uint32_t nb[32];
  float w[32];
};

template <int WPC, int MINB>
__global__ void __launch_bounds__(WPC * 32, MINB) spmm_lean_kernel(SpmmParams p, unsigned* __restrict__ ctr) {
  constexpr int U = 8, F = 256;
  __shared__ __align__(16) SpmmLeanSmem smem[WPC];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  SpmmLeanSmem& sm = smem[w];
  // persistent warps pull items from a counter (largest first): no warp of a CTA idles while
  // its neighbours finish longer rows
  unsigned nxt = lane == 0 ? atomicAdd(ctr, 1u) : 0u;
  for (;;) {
  const int64_t wi = __shfl_sync(0xffffffffu, nxt, 0);
  if (wi >= p.num_items) break;
  if (lane == 0) nxt = atomicAdd(ctr, 1u);
  const Item it = decode_item(p.items, p.off, wi, p.num_split_items, p.chunk);
  const float* xl = p.X + lane * 8;
  float acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.f;
  uint32_t nb = 0;
  float a = 0.f;
  if (it.e0 + lane < it.e1) {
    nb = __ldcs(p.nbr + it.e0 + lane);
    a = p.w ? __ldg(p.w + __ldcs(p.eid + it.e0 + lane)) : 1.f;
  }
  for (uint64_t base = it.e0; base < it.e1; base += 32) {
    const int n = (int)min((uint64_t)32, it.e1 - base);
    const uint32_t nb_last = __shfl_sync(0xffffffffu, nb, n - 1);
    sm.nb[lane] = lane < n ? nb : nb_last;  // rows past n repeat the last one with weight 0
    sm.w[lane] = lane < n ? a : 0.f;
    __syncwarp();
    const uint64_t nx = base + 32 + lane;
    const bool has_next = nx < it.e1;
    const uint32_t nb_n = has_next ? __ldcs(p.nbr + nx) : 0u;
    const uint32_t eid_n = has_next && p.w ? __ldcs(p.eid + nx) : 0u;
    float a_n = 0.f;
    for (int j = 0;;) {
      float x[U][8];
#pragma unroll
      for (int t = 0; t < U; t += 4) {
        const uint4 id4 = *reinterpret_cast<const uint4*>(sm.nb + j + t);
        const uint32_t ids[4] = {id4.x, id4.y, id4.z, id4.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float* src = xl + (uint64_t)ids[k] * F;
          asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
              : "=f"(x[t + k][0]), "=f"(x[t + k][1]), "=f"(x[t + k][2]), "=f"(x[t + k][3]), "=f"(x[t + k][4]),
                "=f"(x[t + k][5]), "=f"(x[t + k][6]), "=f"(x[t + k][7])
              : "l"(src));
        }
      }
      if (j == 0) a_n = has_next ? (p.w ? __ldg(p.w + eid_n) : 1.f) : 0.f;
#pragma unroll
      for (int t = 0; t < U; t += 4) {
        const float4 wv = *reinterpret_cast<const float4*>(sm.w + j + t);
        const float wa[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = fmaf(wa[k], x[t + k][q], acc[q]);
      }
      j += U;
      if (j >= n) break;
    }
    __syncwarp();
    nb = nb_n;
    a = a_n;
  }
  const int c = lane * 8;
  if (!it.split) {
    float o[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float z = acc[q] + (p.bias ? __ldg(p.bias + c + q) : 0.f);
      o[q] = p.relu ? fmaxf(z, 0.f) : z;
    }
    float4* y = reinterpret_cast<float4*>(p.Y + (int64_t)it.row * F + c);
    __stcs(y, make_float4(o[0], o[1], o[2], o[3]));
    __stcs(y + 1, make_float4(o[4], o[5], o[6], o[7]));
  } else {
    float4* q4 = reinterpret_cast<float4*>(p.part + wi * (int64_t)F + c);
    q4[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    q4[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
  __syncwarp();
  }  // items
}

__global__ void spmm_merge_kernel(SpmmParams p, const uint32_t* __restrict__ split_rows,
                                  const uint32_t* __restrict__ split_first, int64_t num_split_rows) {
  const int64_t sr = blockIdx.x;
  if (sr >= num_split_rows) return;
  const int F = p.cols;
  const uint32_t row = split_rows[sr];
  for (int c = threadIdx.x; c < F; c += blockDim.x) {
    float s = 0.f;
    for (int64_t it = split_first[sr]; it < split_first[sr + 1]; ++it) s += p.part[it * F + c];
    s += p.bias ? p.bias[c] : 0.f;
    p.Y[(int64_t)row * F + c] = p.relu ? fmaxf(s, 0.f) : s;
  }
}

// dZ = dOut * [out > 0] (ReLU backward from the stored output) ; db partials per block.
constexpr int kColBlocks = 592;

__global__ void relu_bwd_kernel(int64_t rows, int F, const float* __restrict__ dOut, const float* __restrict__ out,
                                float* __restrict__ dZ, int relu) {
  const int64_t n = rows * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dZ[i] = (!relu || out[i] > 0.f) ? dOut[i] : 0.f;
}

__global__ void colsum_partial_kernel(int64_t rows, int F, const float* __restrict__ X, float* __restrict__ part) {
  const int c = blockIdx.y * blockDim.x + threadIdx.x;
  if (c >= F) return;
  const int64_t per = ceil_div(rows, (int64_t)gridDim.x);
  const int64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  float s = 0.f;
  for (int64_t r = r0; r < r1; ++r) s += __ldg(X + r * F + c);
  part[(int64_t)blockIdx.x * F + c] = s;
}

__global__ void colsum_final_kernel(int nb, int F, const float* __restrict__ part, float* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= F) return;
  float s = 0.f;
  for (int b = 0; b < nb; ++b) s += part[(int64_t)b * F + c];
  out[c] = s;
}

// w[e] = 1 / sqrt(max(1, in_deg(dst e)) * max(1, out_deg(src e)))   (symmetric GCN normalisation)
__global__ void gcn_norm_kernel(int64_t E, const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                                const uint64_t* __restrict__ doff, const uint64_t* __restrict__ soff,
                                float* __restrict__ w) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t u = src[e], v = dst[e];
    const double din = (double)max((uint64_t)1, doff[v + 1] - doff[v]);
    const double dout = (double)max((uint64_t)1, soff[u + 1] - soff[u]);
    w[e] = (float)(1.0 / sqrt(din * dout));
  }
}

// Launch shape, chosen by measurement on B200 (env overrides for experiments):
//   GNNCG_SPMM_OCC = CTAs of 256 threads per SM the kernel is built for (2 | 4 | 8)
//   GNNCG_SPMM_NV  = float-vectors per lane per column slice (1 | 2 | 4 | 8); narrower slices
//                    put more warps on one row, each with fewer registers.
struct SpmmShape {
  int occ, nv;
};

SpmmShape spmm_shape() {
  static const SpmmShape s = [] {
    SpmmShape r{4, 8};
    if (const char* e = getenv("GNNCG_SPMM_OCC")) r.occ = atoi(e);
    if (const char* e = getenv("GNNCG_SPMM_NV")) r.nv = atoi(e);
    if (r.occ != 2 && r.occ != 8) r.occ = 4;
    if (r.nv != 1 && r.nv != 2 && r.nv != 4) r.nv = 8;
    return r;
  }();
  return s;
}

// GNNCG_SPMM_LEAN=0: the general kernel for 256-column rows too (A/B)
bool spmm_lean_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("GNNCG_SPMM_LEAN");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <int VW, int OCC>
int launch_spmm_occ(SpmmParams p, dim3 grid, int max_nv, cudaStream_t s) {
  // split the columns into the fewest slices of <= max_nv vectors per lane, evenly
  const int vecs = p.cols / VW, slices = (int)ceil_div(vecs, 32 * max_nv), per = (int)ceil_div(vecs, slices);
  p.tile = per * VW;
  grid.y = (unsigned)slices;
  const int nvec = (int)ceil_div(per, 32);
  if (nvec <= 1) spmm_kernel<VW, 1, OCC><<<grid, THREADS, 0, s>>>(p);
  else if (nvec <= 2) spmm_kernel<VW, 2, OCC><<<grid, THREADS, 0, s>>>(p);
  else if (nvec <= 4) spmm_kernel<VW, 4, OCC><<<grid, THREADS, 0, s>>>(p);
  else spmm_kernel<VW, 8, OCC><<<grid, THREADS, 0, s>>>(p);
  return GNNCG_OK;
}

template <int VW>
int launch_spmm(const SpmmParams& p, dim3 grid, cudaStream_t s) {
  const SpmmShape sh = spmm_shape();
  if (sh.occ == 8) return launch_spmm_occ<VW, 8>(p, grid, std::min(sh.nv, 2), s);
  if (sh.occ == 2) return launch_spmm_occ<VW, 2>(p, grid, sh.nv, s);
  return launch_spmm_occ<VW, 4>(p, grid, sh.nv, s);
}

}  // namespace
}  // namespace gnncg_b200

using namespace gnncg_b200;

extern "C" {

size_t gnncg_spmm_workspace(const gnncg_sched_t* sched, int cols) {
  // split-row partials, + the lean kernel's work counter
  return sched ? align_up((size_t)sched->num_split_items * cols * sizeof(float)) + 256 : 0;
}

int gnncg_spmm(const gnncg_index_t* idx, const gnncg_sched_t* sched, int cols, const float* edge_w, const float* X,
               const float* bias, int relu, float* Y, void* ws, size_t ws_bytes, void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(idx && sched && cols >= 1, GNNCG_ERR_ARG, "spmm: bad argument");
  GNNCG_REQUIRE(sched->chunk >= 32, GNNCG_ERR_ARG, "spmm: schedule chunk < 32");
  if (sched->num_items == 0) return GNNCG_OK;
  GNNCG_REQUIRE(idx->off && X && Y && sched->items && (idx->num_edges == 0 || idx->nbr), GNNCG_ERR_ARG,
                "spmm: null pointer");
  GNNCG_REQUIRE(!edge_w || idx->num_edges == 0 || idx->eid, GNNCG_ERR_ARG,
                "spmm: edge weights need the index's eid array");
  const size_t need = gnncg_spmm_workspace(sched, cols);
  GNNCG_REQUIRE(ws_bytes >= need && (need == 0 || ws), GNNCG_ERR_WORKSPACE, "spmm: workspace %zu < %zu", ws_bytes,
                need);
  SpmmParams p{idx->off, idx->nbr, idx->eid, sched->items, sched->num_items, sched->num_split_items, sched->chunk,
               cols, 0, edge_w, X, bias, Y, static_cast<float*>(ws), relu};
  cudaStream_t s = as_stream(stream);
  if (cols == 256 && spmm_lean_enabled() && ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & 31) == 0) {
    // 256-column rows (32-byte aligned): the lean kernel, 8 warps x 4 CTAs per SM (64 registers)
#ifndef GNNCG_SPMM_LEAN_WPC
#define GNNCG_SPMM_LEAN_WPC 8
#endif
#ifndef GNNCG_SPMM_LEAN_MINB
#define GNNCG_SPMM_LEAN_MINB 4
#endif
    constexpr int W = GNNCG_SPMM_LEAN_WPC, M = GNNCG_SPMM_LEAN_MINB;
    p.tile = 256;
    unsigned* ctr = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + align_up((size_t)sched->num_split_items * cols * sizeof(float)));
    GNNCG_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(unsigned), s));
    const L2Window win = l2_window(sched, X, 256 * sizeof(float));
    int sms = 148;
    {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const dim3 g((unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(sched->num_items, W), (int64_t)sms * M)));
    if (win.bytes == 0) {
      spmm_lean_kernel<W, M><<<g, W * 32, 0, s>>>(p, ctr);
    } else {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = g;
      cfg.blockDim = dim3(W * 32);
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeAccessPolicyWindow;
      at[0].val.accessPolicyWindow.base_ptr = const_cast<void*>(win.base);
      at[0].val.accessPolicyWindow.num_bytes = win.bytes;
      at[0].val.accessPolicyWindow.hitRatio = 1.0f;
      at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, spmm_lean_kernel<W, M>, p, ctr);
    }
  } else {
    dim3 grid((unsigned)ceil_div(sched->num_items, WARPS));
    int rc = cols % 4 == 0 ? launch_spmm<4>(p, grid, s) : (cols % 2 == 0 ? launch_spmm<2>(p, grid, s)
                                                                           : launch_spmm<1>(p, grid, s));
    if (rc) return rc;
  }
  GNNCG_LAUNCH_CHECK();
  if (sched->num_split_rows > 0) {
    spmm_merge_kernel<<<(unsigned)sched->num_split_rows, 256, 0, s>>>(p, sched->split_rows, sched->split_first,
                                                                    sched->num_split_rows);
    GNNCG_LAUNCH_CHECK();
  }
  return GNNCG_OK;
}

size_t gnncg_relu_bwd_workspace(int cols) { return align_up((size_t)kColBlocks * cols * sizeof(float)); }

int gnncg_relu_bwd(int64_t rows, int cols, const float* dOut, const float* out, int relu, float* dZ, float* dbias,
                   void* ws, size_t ws_bytes, void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(rows >= 0 && cols >= 1, GNNCG_ERR_SHAPE, "relu_bwd: bad shape");
  GNNCG_REQUIRE(dOut && dZ && (!relu || out), GNNCG_ERR_ARG, "relu_bwd: null pointer");
  cudaStream_t s = as_stream(stream);
  if (rows > 0) {
    relu_bwd_kernel<<<(unsigned)std::min<int64_t>(ceil_div(rows * cols, 256), 148 * 16), 256, 0, s>>>(
        rows, cols, dOut, out, dZ, relu);
    GNNCG_LAUNCH_CHECK();
  }
  if (dbias) {
    GNNCG_REQUIRE(ws && ws_bytes >= gnncg_relu_bwd_workspace(cols), GNNCG_ERR_WORKSPACE, "relu_bwd: workspace");
    float* part = static_cast<float*>(ws);
    dim3 g1(kColBlocks, (unsigned)ceil_div(cols, 256));
    colsum_partial_kernel<<<g1, 256, 0, s>>>(rows, cols, dZ, part);
    GNNCG_LAUNCH_CHECK();
    colsum_final_kernel<<<(unsigned)ceil_div(cols, 256), 256, 0, s>>>(kColBlocks, cols, part, dbias);
    GNNCG_LAUNCH_CHECK();
  }
  return GNNCG_OK;
}

int gnncg_gcn_norm(int64_t num_edges, const uint32_t* edge_src, const uint32_t* edge_dst, const gnncg_index_t* csr_dst,
                   const gnncg_index_t* csc_src, float* w, void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(csr_dst && csc_src && (num_edges == 0 || (edge_src && edge_dst && w)), GNNCG_ERR_ARG,
                "gcn_norm: null pointer");
  if (num_edges == 0) return GNNCG_OK;
  gcn_norm_kernel<<<(unsigned)std::min<int64_t>(ceil_div(num_edges, 256), 148 * 16), 256, 0, as_stream(stream)>>>(
      num_edges, edge_src, edge_dst, csr_dst->off, csc_src->off, w);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

}  // extern "C"
