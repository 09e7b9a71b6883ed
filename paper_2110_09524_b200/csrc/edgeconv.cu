// SPDX-License-Identifier: Apache-2.0
//
// EdgeConv fused region (K6) and its argmax-routing backward (K7).
//   reorganized form: Th = H Theta, Ph = H Phi run
//   once per vertex (dense GEMM), then per destination v
//     out[v,c] = max_{(u,e) in in(v)} ((Th[u,c] - Th[v,c]) + Ph[v,c])
//   with the lowest-edge-id maximiser recorded and 0 / 0xFFFFFFFF
//   for empty rows.  Only the O(|V| C) argmax is stashed
//   (PAPER.md:409).
// Bit-exact argmax: the expression is evaluated exactly as written in fp32
// round-to-nearest (__fsub_rn/__fadd_rn: no contraction or reassociation) and
// compared with a strict '>' walking the row in edge-id order -- the same
// arithmetic as oracle/oracle.cpp:edgeconv_fwd.
#include "common.cuh"

namespace gnncg_b200 {
namespace {

constexpr uint32_t kNoEdge = 0xFFFFFFFFu;

template <int VW>
struct Vec;
template <>
struct Vec<1> { using F = float; using U = uint32_t; };
template <>
struct Vec<2> { using F = float2; using U = uint2; };
template <>
struct Vec<4> { using F = float4; using U = uint4; };

template <int VW>
__device__ __forceinline__ void ldv(const float* p, float (&x)[VW]) {
  constexpr int W = VW < 4 ? VW : 4;
#pragma unroll
  for (int k = 0; k < VW / W; ++k) {
    const typename Vec<W>::F t = __ldg(reinterpret_cast<const typename Vec<W>::F*>(p) + k);
    const float* q = reinterpret_cast<const float*>(&t);
#pragma unroll
    for (int i = 0; i < W; ++i) x[k * W + i] = q[i];
  }
}
template <int VW>
__device__ __forceinline__ void ldv(const uint32_t* p, uint32_t (&x)[VW]) {
  constexpr int W = VW < 4 ? VW : 4;
#pragma unroll
  for (int k = 0; k < VW / W; ++k) {
    const typename Vec<W>::U t = __ldg(reinterpret_cast<const typename Vec<W>::U*>(p) + k);
    const uint32_t* q = reinterpret_cast<const uint32_t*>(&t);
#pragma unroll
    for (int i = 0; i < W; ++i) x[k * W + i] = q[i];
  }
}
template <int VW, typename T>
__device__ __forceinline__ void stv(T* p, const T (&x)[VW]) {
#pragma unroll
  for (int i = 0; i < VW; ++i) p[i] = x[i];
}

// K6: warp per destination row, VW consecutive columns per lane (32 VW columns per pass).  The
// row's neighbour and edge ids are read 32 at a time (one coalesced load each) and broadcast by
// shuffles; rows are gathered 4 edges ahead.  Edges are walked in the row's (edge-id) order.
template <int VW>
__global__ void __launch_bounds__(256) edgeconv_fwd_kernel(int64_t rows, int C, int64_t row_base,
                                                           const uint64_t* __restrict__ off,
                                                           const uint32_t* __restrict__ nbr,
                                                           const uint32_t* __restrict__ eid,
                                                           const float* __restrict__ Th, int64_t ldt,
                                                           const float* __restrict__ Ph, int64_t ldp,
                                                           float* __restrict__ out, uint32_t* __restrict__ amax) {
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const uint64_t e0 = off[r], e1 = off[r + 1];
  const int64_t v = row_base + r;
  for (int c0 = 0; c0 < C; c0 += 32 * VW) {
    const int c = c0 + lane * VW;
    const bool on = c < C;
    float best[VW], thv[VW], phv[VW];
    uint32_t arg[VW];
#pragma unroll
    for (int i = 0; i < VW; ++i) { best[i] = 0.f; arg[i] = kNoEdge; thv[i] = 0.f; phv[i] = 0.f; }
    if (on && e0 < e1) {
      ldv<VW>(Th + v * ldt + c, thv);
      ldv<VW>(Ph + r * ldp + c, phv);
    }
    for (uint64_t base = e0; base < e1; base += 32) {
      const int n = (int)min((uint64_t)32, e1 - base);
      const uint32_t my_u = lane < n ? __ldg(nbr + base + lane) : 0u;
      const uint32_t my_e = lane < n ? __ldg(eid + base + lane) : 0u;
      for (int j = 0; j < n; j += U) {
        float x[U][VW];
#pragma unroll
        for (int t = 0; t < U; ++t) {
          const uint32_t u = __shfl_sync(0xffffffffu, my_u, (j + t) & 31);
          if (on && j + t < n) ldv<VW>(Th + (int64_t)u * ldt + c, x[t]);
        }
#pragma unroll
        for (int t = 0; t < U; ++t) {
          const uint32_t id = __shfl_sync(0xffffffffu, my_e, (j + t) & 31);
          if (j + t < n) {
#pragma unroll
            for (int i = 0; i < VW; ++i) {
              const float val = __fadd_rn(__fsub_rn(x[t][i], thv[i]), phv[i]);
              if (arg[i] == kNoEdge || val > best[i]) { best[i] = val; arg[i] = id; }
            }
          }
        }
      }
    }
    if (on) {
      stv<VW>(out + r * C + c, best);
      stv<VW>(amax + r * C + c, arg);
    }
  }
}

// K7: inverse-argmax gather over csc_src (deterministic, atomic-free): for each out-edge (u, e, v)
// of source u, column c takes g[v, c] iff amax[v, c] == e.  VW columns per lane.  EAGER (the
// default; GNNCG_EC_EAGER=0 for the other) loads g with amax instead of after a match: one
// dependent round trip per 4 edges instead of two, for bytes that are L2-resident here
// (C3, k = 40: 0.138 vs 0.147 ms per launch).
template <int VW, bool EAGER>
__global__ void __launch_bounds__(256) edgeconv_bwd_kernel(int64_t rows, int C, const uint64_t* __restrict__ soff,
                                                           const uint32_t* __restrict__ snbr,
                                                           const uint32_t* __restrict__ seid,
                                                           const uint64_t* __restrict__ doff,
                                                           const uint32_t* __restrict__ amax,
                                                           const float* __restrict__ g, float* __restrict__ dTh,
                                                           int64_t ldt, float* __restrict__ dPh, int64_t ldp) {
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  const int64_t u = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (u >= rows) return;
  const uint64_t e0 = soff[u], e1 = soff[u + 1];
  const bool has_in = doff[u + 1] > doff[u];
  for (int c0 = 0; c0 < C; c0 += 32 * VW) {
    const int c = c0 + lane * VW;
    const bool on = c < C;
    float acc[VW];
#pragma unroll
    for (int i = 0; i < VW; ++i) acc[i] = 0.f;
    for (uint64_t base = e0; base < e1; base += 32) {
      const int n = (int)min((uint64_t)32, e1 - base);
      const uint32_t my_v = lane < n ? __ldg(snbr + base + lane) : 0u;
      const uint32_t my_e = lane < n ? __ldg(seid + base + lane) : 0u;
      for (int j = 0; j < n; j += U) {
        uint32_t am[U][VW];
        float gv[U][VW];
        int64_t vv[U];
#pragma unroll
        for (int t = 0; t < U; ++t) {
          vv[t] = __shfl_sync(0xffffffffu, my_v, (j + t) & 31);
          if (on && j + t < n) {
            ldv<VW>(amax + vv[t] * C + c, am[t]);
            if (EAGER) ldv<VW>(g + vv[t] * C + c, gv[t]);
          }
        }
#pragma unroll
        for (int t = 0; t < U; ++t) {
          const uint32_t id = __shfl_sync(0xffffffffu, my_e, (j + t) & 31);
          if (on && j + t < n) {
            if (!EAGER) {
              bool any = false;
#pragma unroll
              for (int i = 0; i < VW; ++i) any |= am[t][i] == id;
              if (any) ldv<VW>(g + vv[t] * C + c, gv[t]);
            }
#pragma unroll
            for (int i = 0; i < VW; ++i)
              if (am[t][i] == id) acc[i] += gv[t][i];
          }
        }
      }
    }
    if (on) {
      float gu[VW], dt[VW];
#pragma unroll
      for (int i = 0; i < VW; ++i) gu[i] = 0.f;
      if (has_in) ldv<VW>(g + u * C + c, gu);
#pragma unroll
      for (int i = 0; i < VW; ++i) dt[i] = acc[i] - gu[i];
      stv<VW>(dTh + u * ldt + c, dt);
      stv<VW>(dPh + u * ldp + c, gu);
    }
  }
}

// Column vector width: 4 / 2 floats per lane when every row start is 16 / 8-byte aligned.  (8 per
// lane, one pass at C = 256: 119-128 registers, no faster than two passes of 4.)
template <int VW, bool EAGER>
void launch_bwd(unsigned grid, void* stream, const gnncg_index_t* csc, const gnncg_index_t* csr, int C,
                const uint32_t* amax, const float* g, float* dTh, int64_t ldt, float* dPh, int64_t ldp) {
  edgeconv_bwd_kernel<VW, EAGER><<<grid, 256, 0, as_stream(stream)>>>(csc->num_rows, C, csc->off, csc->nbr, csc->eid,
                                                                     csr->off, amax, g, dTh, ldt, dPh, ldp);
}

bool ec_eager() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("GNNCG_EC_EAGER"); v = e ? atoi(e) : 1; }
  return v == 1;
}

int edge_vw(int C, const void* a, int64_t lda, const void* b, int64_t ldb) {
  auto ok = [&](int w) {
    return C % w == 0 && lda % w == 0 && ldb % w == 0 && ((uintptr_t)a % (4 * w)) == 0 &&
           ((uintptr_t)b % (4 * w)) == 0;
  };
  return ok(4) && C >= 128 ? 4 : ok(2) && C >= 64 ? 2 : 1;
}

}  // namespace
}  // namespace gnncg_b200

using namespace gnncg_b200;

extern "C" {

int gnncg_edgeconv_fwd(const gnncg_index_t* csr, int C, int64_t row_base, const float* Th, int64_t ldt,
                       const float* Ph, int64_t ldp, float* out, uint32_t* amax, void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(csr && C >= 1, GNNCG_ERR_SHAPE, "edgeconv_fwd: bad shape");
  GNNCG_REQUIRE(ldt >= C && ldp >= C && row_base >= 0, GNNCG_ERR_SHAPE, "edgeconv_fwd: leading dimension < C");
  if (csr->num_rows == 0) return GNNCG_OK;
  GNNCG_REQUIRE(csr->off && (csr->num_edges == 0 || (csr->nbr && csr->eid)) && Th && Ph && out && amax, GNNCG_ERR_ARG,
                "edgeconv_fwd: null pointer (csr_dst.eid is required for the argmax)");
  const unsigned grid = (unsigned)ceil_div(csr->num_rows, 8);
  const int vw = edge_vw(C, Th, ldt, Ph, ldp);
#define GNNCG_EC_FWD(W)                                                                                     \
  edgeconv_fwd_kernel<W><<<grid, 256, 0, as_stream(stream)>>>(csr->num_rows, C, row_base, csr->off, csr->nbr, \
                                                              csr->eid, Th, ldt, Ph, ldp, out, amax)
  if (vw == 4) GNNCG_EC_FWD(4);
  else if (vw == 2) GNNCG_EC_FWD(2);
  else GNNCG_EC_FWD(1);
#undef GNNCG_EC_FWD
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

int gnncg_edgeconv_bwd(const gnncg_index_t* csc, const gnncg_index_t* csr, int C, const uint32_t* amax,
                       const float* g, float* dTh, int64_t ldt, float* dPh, int64_t ldp, void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(csc && csr && C >= 1 && ldt >= C && ldp >= C, GNNCG_ERR_SHAPE, "edgeconv_bwd: bad shape");
  GNNCG_REQUIRE(csc->num_rows == csr->num_rows, GNNCG_ERR_SHAPE, "edgeconv_bwd: csc/csr row mismatch");
  if (csc->num_rows == 0) return GNNCG_OK;
  GNNCG_REQUIRE(csc->off && (csc->num_edges == 0 || (csc->nbr && csc->eid)) && csr->off && amax && g && dTh && dPh,
                GNNCG_ERR_ARG,
                "edgeconv_bwd: null pointer (csc_src.eid is required)");
  const unsigned grid = (unsigned)ceil_div(csc->num_rows, 8);
  // (amax and g are dense C-wide rows: their alignment follows from C and the base pointers)
  int vw = edge_vw(C, dTh, ldt, dPh, ldp);
  while (vw > 1 && (((uintptr_t)amax % (4 * std::min(vw, 4))) || ((uintptr_t)g % (4 * std::min(vw, 4))))) vw /= 2;
#define GNNCG_EC_BWD(W)                                                                                      \
  (ec_eager() ? launch_bwd<W, true>(grid, stream, csc, csr, C, amax, g, dTh, ldt, dPh, ldp)                     \
              : launch_bwd<W, false>(grid, stream, csc, csr, C, amax, g, dTh, ldt, dPh, ldp))
  if (vw == 4) GNNCG_EC_BWD(4);
  else if (vw == 2) GNNCG_EC_BWD(2);
  else GNNCG_EC_BWD(1);
#undef GNNCG_EC_BWD
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

}  // extern "C"
