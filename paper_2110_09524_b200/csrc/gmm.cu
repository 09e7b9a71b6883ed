// SPDX-License-Identifier: Apache-2.0
//
// GMMConv / MoNet fused region (K8), forward and recompute backward.
//   PAPER.md:591-605 ; SPEC.md:216 (diagonal Sigma).  Parameterisation (recorded
//   in DESIGN.md): Sigma_k^{-1} = diag(sinv_k^2), sinv learned.
//   Reorganized: one dense GEMM Y = H [W | P_l | P_r] gives hW, pl, pr per vertex;
//   the pseudo-coordinate of edge (u,e,v) is m = pl[u] + pr[v] (u_add_v).
//     w_k = exp(-1/2 sum_t (m_t - mu_kt)^2 sinv_kt^2)
//     out[v,:] = (1/K) sum_e sum_k w_k hW[u,k,:]
// Backward (recompute; nothing O(|E|) stashed):
//   pass 1 over csr_dst: d pr[v], and per-row partials of dmu / dsinv (merged in
//     row order -> deterministic);
//   pass 2 over csc_src: d hW[u,k,:] = (1/K) sum_e w_k dOut[v], d pl[u].
#include <cfloat>

#include "common.cuh"

namespace gnncg_b200 {
namespace {

constexpr int MAXK = 8, MAXR = 4, MAXKF = 256, WARPS = 8;

struct GmmSmem {
  uint32_t nb[32];
  float w[32 * (MAXK + 1)];
  float red[MAXKF];
  float row[MAXKF];
};

struct GmmArgs {
  int64_t rows;
  int K, r, f;
  const uint64_t* off;
  const uint32_t* nbr;
  const float* Y;
  int64_t ldy;
  const float *mu, *sinv, *dOut;
  float *out, *dY, *part;
};

__device__ __forceinline__ void gauss(const GmmArgs& a, const float* pl_u, const float* pr_v, float (&w)[MAXK],
                                      float (&md)[MAXK][MAXR]) {
#pragma unroll
  for (int k = 0; k < MAXK; ++k) {
    float q = 0.f;
#pragma unroll
    for (int t = 0; t < MAXR; ++t) {
      if (k < a.K && t < a.r) {
        const float x = pl_u[t] + pr_v[t] - __ldg(a.mu + k * a.r + t);
        const float s = __ldg(a.sinv + k * a.r + t);
        md[k][t] = x;
        q = fmaf(x * x, s * s, q);
      } else {
        md[k][t] = 0.f;
      }
    }
    w[k] = k < a.K ? __expf(-0.5f * q) : 0.f;
  }
}

__global__ void __launch_bounds__(256) gmm_fwd_kernel(GmmArgs a) {
  __shared__ GmmSmem smem[WARPS];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  GmmSmem& sm = smem[wid];
  const int64_t v = (int64_t)blockIdx.x * WARPS + wid;
  if (v >= a.rows) return;
  const int K = a.K, r = a.r, f = a.f, Kf = K * f;
  float prv[MAXR];
#pragma unroll
  for (int t = 0; t < MAXR; ++t) prv[t] = t < r ? __ldg(a.Y + v * a.ldy + Kf + r + t) : 0.f;
  float acc[MAXKF / 32];
#pragma unroll
  for (int i = 0; i < MAXKF / 32; ++i) acc[i] = 0.f;
  const uint64_t e0 = a.off[v], e1 = a.off[v + 1];
  for (uint64_t base = e0; base < e1; base += 32) {
    const int n = (int)min((uint64_t)32, e1 - base);
    if (lane < n) {
      const uint32_t u = __ldg(a.nbr + base + lane);
      sm.nb[lane] = u;
      float plu[MAXR];
#pragma unroll
      for (int t = 0; t < MAXR; ++t) plu[t] = t < r ? __ldg(a.Y + (int64_t)u * a.ldy + Kf + t) : 0.f;
      float w[MAXK], md[MAXK][MAXR];
      gauss(a, plu, prv, w, md);
#pragma unroll
      for (int k = 0; k < MAXK; ++k)
        if (k < K) sm.w[lane * (MAXK + 1) + k] = w[k];
    }
    __syncwarp();
    for (int j = 0; j < n; ++j) {
      const float* y = a.Y + (int64_t)sm.nb[j] * a.ldy;
#pragma unroll
      for (int i = 0; i < MAXKF / 32; ++i) {
        const int c = i * 32 + lane;
        if (c < Kf) acc[i] = fmaf(sm.w[j * (MAXK + 1) + c / f], __ldg(y + c), acc[i]);
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int i = 0; i < MAXKF / 32; ++i) {
    const int c = i * 32 + lane;
    if (c < Kf) sm.red[c] = acc[i];
  }
  __syncwarp();
  const float invK = 1.f / (float)K;
  for (int c = lane; c < f; c += 32) {
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += sm.red[k * f + c];
    a.out[v * f + c] = s * invK;
  }
}

// pass 1 over csr_dst: lane per edge.
__global__ void __launch_bounds__(256) gmm_bwd_dst_kernel(GmmArgs a) {
  __shared__ GmmSmem smem[WARPS];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  GmmSmem& sm = smem[wid];
  const int64_t v = (int64_t)blockIdx.x * WARPS + wid;
  if (v >= a.rows) return;
  const int K = a.K, r = a.r, f = a.f, Kf = K * f;
  const float invK = 1.f / (float)K;
  for (int c = lane; c < f; c += 32) sm.row[c] = __ldg(a.dOut + v * f + c);
  __syncwarp();
  float prv[MAXR], dpr[MAXR], dmu[MAXK][MAXR], dsi[MAXK][MAXR];
#pragma unroll
  for (int t = 0; t < MAXR; ++t) {
    prv[t] = t < r ? __ldg(a.Y + v * a.ldy + Kf + r + t) : 0.f;
    dpr[t] = 0.f;
#pragma unroll
    for (int k = 0; k < MAXK; ++k) { dmu[k][t] = 0.f; dsi[k][t] = 0.f; }
  }
  const uint64_t e0 = a.off[v], e1 = a.off[v + 1];
  for (uint64_t e = e0 + lane; e < e1; e += 32) {
    const int64_t u = __ldg(a.nbr + e);
    const float* y = a.Y + u * a.ldy;
    float plu[MAXR];
#pragma unroll
    for (int t = 0; t < MAXR; ++t) plu[t] = t < r ? __ldg(y + Kf + t) : 0.f;
    float w[MAXK], md[MAXK][MAXR];
    gauss(a, plu, prv, w, md);
#pragma unroll
    for (int k = 0; k < MAXK; ++k) {
      if (k < K) {
        float dw = 0.f;
        for (int c = 0; c < f; ++c) dw = fmaf(sm.row[c], __ldg(y + k * f + c), dw);
        const float dq = -0.5f * w[k] * dw * invK;
#pragma unroll
        for (int t = 0; t < MAXR; ++t) {
          if (t < r) {
            const float s = __ldg(a.sinv + k * r + t), x = md[k][t];
            const float dmd = dq * 2.f * x * s * s;
            dsi[k][t] = fmaf(dq * 2.f * x * x, s, dsi[k][t]);
            dmu[k][t] -= dmd;
            dpr[t] += dmd;
          }
        }
      }
    }
  }
  float* part = a.part + v * (int64_t)(2 * K * r);
#pragma unroll
  for (int t = 0; t < MAXR; ++t) {
    if (t < r) {
      const float s = warp_sum(dpr[t]);
      if (lane == 0) a.dY[v * a.ldy + Kf + r + t] = s;
#pragma unroll
      for (int k = 0; k < MAXK; ++k) {
        if (k < K) {
          const float m1 = warp_sum(dmu[k][t]);
          const float s1 = warp_sum(dsi[k][t]);
          if (lane == 0) { part[k * r + t] = m1; part[K * r + k * r + t] = s1; }
        }
      }
    }
  }
}

// pass 2 over csc_src.
__global__ void __launch_bounds__(256) gmm_bwd_src_kernel(GmmArgs a) {
  __shared__ GmmSmem smem[WARPS];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  GmmSmem& sm = smem[wid];
  const int64_t u = (int64_t)blockIdx.x * WARPS + wid;
  if (u >= a.rows) return;
  const int K = a.K, r = a.r, f = a.f, Kf = K * f;
  const float invK = 1.f / (float)K;
  const float* yu = a.Y + u * a.ldy;
  for (int c = lane; c < Kf; c += 32) sm.row[c] = __ldg(yu + c);
  float plu[MAXR], dpl[MAXR];
#pragma unroll
  for (int t = 0; t < MAXR; ++t) { plu[t] = t < r ? __ldg(yu + Kf + t) : 0.f; dpl[t] = 0.f; }
  __syncwarp();
  float acc[MAXKF / 32];
#pragma unroll
  for (int i = 0; i < MAXKF / 32; ++i) acc[i] = 0.f;
  const uint64_t e0 = a.off[u], e1 = a.off[u + 1];
  for (uint64_t base = e0; base < e1; base += 32) {
    const int n = (int)min((uint64_t)32, e1 - base);
    if (lane < n) {
      const int64_t v = __ldg(a.nbr + base + lane);
      sm.nb[lane] = (uint32_t)v;
      float prv[MAXR];
#pragma unroll
      for (int t = 0; t < MAXR; ++t) prv[t] = t < r ? __ldg(a.Y + v * a.ldy + Kf + r + t) : 0.f;
      float w[MAXK], md[MAXK][MAXR];
      gauss(a, plu, prv, w, md);
      const float* g = a.dOut + v * f;
#pragma unroll
      for (int k = 0; k < MAXK; ++k) {
        if (k < K) {
          sm.w[lane * (MAXK + 1) + k] = w[k] * invK;
          float dw = 0.f;
          for (int c = 0; c < f; ++c) dw = fmaf(__ldg(g + c), sm.row[k * f + c], dw);
          const float dq = -0.5f * w[k] * dw * invK;
#pragma unroll
          for (int t = 0; t < MAXR; ++t)
            if (t < r) {
              const float s = __ldg(a.sinv + k * r + t);
              dpl[t] = fmaf(dq * 2.f * md[k][t], s * s, dpl[t]);
            }
        }
      }
    }
    __syncwarp();
    for (int j = 0; j < n; ++j) {
      const float* g = a.dOut + (int64_t)sm.nb[j] * f;
#pragma unroll
      for (int i = 0; i < MAXKF / 32; ++i) {
        const int c = i * 32 + lane;
        if (c < Kf) acc[i] = fmaf(sm.w[j * (MAXK + 1) + c / f], __ldg(g + c % f), acc[i]);
      }
    }
    __syncwarp();
  }
  float* dy = a.dY + u * a.ldy;
#pragma unroll
  for (int i = 0; i < MAXKF / 32; ++i) {
    const int c = i * 32 + lane;
    if (c < Kf) dy[c] = acc[i];
  }
#pragma unroll
  for (int t = 0; t < MAXR; ++t) {
    if (t < r) {
      const float s = warp_sum(dpl[t]);
      if (lane == 0) dy[Kf + t] = s;
    }
  }
}

// dmu / dsinv = sum over rows of the per-row partials, in row order.
__global__ void gmm_param_reduce_kernel(int64_t rows, int n, const float* __restrict__ part, float* __restrict__ dmu,
                                        float* __restrict__ dsinv, int Kr) {
  // one warp per parameter entry; lanes stride rows, then a fixed-order tree.
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= n) return;
  float s = 0.f;
  for (int64_t rr = lane; rr < rows; rr += 32) s += part[rr * n + q];
  s = warp_sum(s);
  if (lane == 0) {
    if (q < Kr) dmu[q] = s; else dsinv[q - Kr] = s;
  }
}

int check(const gnncg_index_t* idx, int K, int r, int f, int64_t ldy) {
  GNNCG_REQUIRE(idx, GNNCG_ERR_ARG, "gmm: null index");
  GNNCG_REQUIRE(K >= 1 && K <= MAXK && r >= 1 && r <= MAXR && f >= 1 && K * f <= MAXKF, GNNCG_ERR_UNSUPPORTED,
                "gmm: (K=%d, r=%d, f=%d) outside compiled limits K<=%d r<=%d K*f<=%d", K, r, f, MAXK, MAXR, MAXKF);
  GNNCG_REQUIRE(ldy >= (int64_t)K * f + 2 * r, GNNCG_ERR_SHAPE, "gmm: ldy < K*f + 2r");
  return GNNCG_OK;
}

}  // namespace
}  // namespace gnncg_b200

using namespace gnncg_b200;

extern "C" {

int gnncg_gmm_fwd(const gnncg_index_t* csr, int K, int r, int f, const float* Y, int64_t ldy, const float* mu,
                  const float* sinv, float* out, void* stream) {
  GNNCG_DEVICE_GUARD();
  int rc = check(csr, K, r, f, ldy);
  if (rc) return rc;
  if (csr->num_rows == 0) return GNNCG_OK;
  GNNCG_REQUIRE(csr->off && (csr->num_edges == 0 || csr->nbr) && Y && mu && sinv && out, GNNCG_ERR_ARG,
                "gmm_fwd: null pointer");
  GmmArgs a{csr->num_rows, K, r, f, csr->off, csr->nbr, Y, ldy, mu, sinv, nullptr, out, nullptr, nullptr};
  gmm_fwd_kernel<<<(unsigned)ceil_div(csr->num_rows, WARPS), 256, 0, as_stream(stream)>>>(a);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

size_t gnncg_gmm_bwd_workspace(const gnncg_index_t* csr, int K, int r) {
  return csr ? align_up((size_t)csr->num_rows * 2 * K * r * sizeof(float)) : 0;
}

int gnncg_gmm_bwd(const gnncg_index_t* csr, const gnncg_index_t* csc, int K, int r, int f, const float* Y,
                  int64_t ldy, const float* mu, const float* sinv, const float* dOut, float* dY, float* dmu,
                  float* dsinv, void* ws, size_t ws_bytes, void* stream) {
  GNNCG_DEVICE_GUARD();
  int rc = check(csr, K, r, f, ldy);
  if (rc) return rc;
  GNNCG_REQUIRE(csc && csc->num_rows == csr->num_rows, GNNCG_ERR_SHAPE, "gmm_bwd: csc/csr row mismatch");
  GNNCG_REQUIRE(dmu && dsinv, GNNCG_ERR_ARG, "gmm_bwd: null pointer");
  const size_t need = gnncg_gmm_bwd_workspace(csr, K, r);
  GNNCG_REQUIRE(ws_bytes >= need && (need == 0 || ws), GNNCG_ERR_WORKSPACE, "gmm_bwd: workspace %zu < %zu",
                ws_bytes, need);
  cudaStream_t s = as_stream(stream);
  if (csr->num_rows == 0) {
    GNNCG_CUDA_TRY(cudaMemsetAsync(dmu, 0, sizeof(float) * K * r, s));
    GNNCG_CUDA_TRY(cudaMemsetAsync(dsinv, 0, sizeof(float) * K * r, s));
    return GNNCG_OK;
  }
  GNNCG_REQUIRE(csr->off && csc->off && (csr->num_edges == 0 || (csr->nbr && csc->nbr)) && Y && mu && sinv && dOut &&
                    dY,
                GNNCG_ERR_ARG,
                "gmm_bwd: null pointer");
  GmmArgs a{csr->num_rows, K, r, f, csr->off, csr->nbr, Y, ldy, mu, sinv, dOut, nullptr, dY,
            static_cast<float*>(ws)};
  const unsigned grid = (unsigned)ceil_div(csr->num_rows, WARPS);
  gmm_bwd_dst_kernel<<<grid, 256, 0, s>>>(a);
  GNNCG_LAUNCH_CHECK();
  a.off = csc->off;
  a.nbr = csc->nbr;
  gmm_bwd_src_kernel<<<grid, 256, 0, s>>>(a);
  GNNCG_LAUNCH_CHECK();
  const int n = 2 * K * r;
  gmm_param_reduce_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, s>>>(csr->num_rows, n, a.part, dmu, dsinv, K * r);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

}  // extern "C"
