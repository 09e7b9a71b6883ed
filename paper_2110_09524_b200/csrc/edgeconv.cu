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

__global__ void __launch_bounds__(256) edgeconv_fwd_kernel(int64_t rows, int C, int64_t row_base,
                                                           const uint64_t* __restrict__ off,
                                                           const uint32_t* __restrict__ nbr,
                                                           const uint32_t* __restrict__ eid,
                                                           const float* __restrict__ Th, int64_t ldt,
                                                           const float* __restrict__ Ph, int64_t ldp,
                                                           float* __restrict__ out, uint32_t* __restrict__ amax) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const uint64_t e0 = off[r], e1 = off[r + 1];
  const int64_t v = row_base + r;
  for (int c = lane; c < C; c += 32) {
    float best = 0.f;
    uint32_t arg = kNoEdge;
    if (e0 < e1) {
      const float thv = __ldg(Th + v * ldt + c), phv = __ldg(Ph + r * ldp + c);
      uint64_t e = e0;
      for (; e + 4 <= e1; e += 4) {
        float x[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) x[t] = __ldg(Th + (int64_t)__ldg(nbr + e + t) * ldt + c);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float val = __fadd_rn(__fsub_rn(x[t], thv), phv);
          if (arg == kNoEdge || val > best) { best = val; arg = __ldg(eid + e + t); }
        }
      }
      for (; e < e1; ++e) {
        const float val = __fadd_rn(__fsub_rn(__ldg(Th + (int64_t)__ldg(nbr + e) * ldt + c), thv), phv);
        if (arg == kNoEdge || val > best) { best = val; arg = __ldg(eid + e); }
      }
    }
    out[r * C + c] = best;
    amax[r * C + c] = arg;
  }
}

// Inverse-argmax gather over csc_src (deterministic, atomic-free).
__global__ void __launch_bounds__(256) edgeconv_bwd_kernel(int64_t rows, int C, const uint64_t* __restrict__ soff,
                                                           const uint32_t* __restrict__ snbr,
                                                           const uint32_t* __restrict__ seid,
                                                           const uint64_t* __restrict__ doff,
                                                           const uint32_t* __restrict__ amax,
                                                           const float* __restrict__ g, float* __restrict__ dTh,
                                                           int64_t ldt, float* __restrict__ dPh, int64_t ldp) {
  const int lane = threadIdx.x & 31;
  const int64_t u = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (u >= rows) return;
  const uint64_t e0 = soff[u], e1 = soff[u + 1];
  const bool has_in = doff[u + 1] > doff[u];
  for (int c = lane; c < C; c += 32) {
    float acc = 0.f;
    for (uint64_t e = e0; e < e1; ++e) {
      const int64_t v = __ldg(snbr + e);
      if (__ldg(amax + v * C + c) == __ldg(seid + e)) acc += __ldg(g + v * C + c);
    }
    const float gu = has_in ? __ldg(g + u * C + c) : 0.f;
    dTh[u * ldt + c] = acc - gu;
    dPh[u * ldp + c] = gu;
  }
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
  edgeconv_fwd_kernel<<<(unsigned)ceil_div(csr->num_rows, 8), 256, 0, as_stream(stream)>>>(
      csr->num_rows, C, row_base, csr->off, csr->nbr, csr->eid, Th, ldt, Ph, ldp, out, amax);
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
  edgeconv_bwd_kernel<<<(unsigned)ceil_div(csc->num_rows, 8), 256, 0, as_stream(stream)>>>(
      csc->num_rows, C, csc->off, csc->nbr, csc->eid, csr->off, amax, g, dTh, ldt, dPh, ldp);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

}  // extern "C"
