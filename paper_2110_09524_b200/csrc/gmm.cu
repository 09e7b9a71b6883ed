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
// CTAs per SM the register allocation must allow (build-time A/B knobs): the backward passes spill
// below 64 registers; the forward takes 48 at 5 CTAs without spilling (C4 step 0.304 -> 0.298 ms,
// profiles/r02_gmm_ab.txt).
#ifndef GNNCG_GMM_MINB
#define GNNCG_GMM_MINB 4
#endif
#ifndef GNNCG_GMM_MINB_FWD
#define GNNCG_GMM_MINB_FWD 5
#endif

struct GmmArgs {
  int64_t rows;
  int K, r, f;
  const uint64_t* off;
  const uint32_t* nbr;
  const float* Y;
  int64_t ldy;
  const float *mu, *sinv, *dOut;
  float *out, *dY, *part;
  bool vec4;  // f % 4 == 0 and 16-byte rows of Y / dOut: the per-edge f loops read float4s
};

// w_k of one edge: exp(-1/2 sum_t (pl_u + pr_v - mu_k)_t^2 sinv_kt^2).  k < K, t < r are runtime
// guards inside fully unrolled loops, so pl / pr stay in registers; nothing of size K x r is
// kept per lane (the earlier per-lane [K][r] arrays cost 174-216 registers: 8 warps per SM).
__device__ __forceinline__ float gmm_w(const GmmArgs& a, int k, const float (&plu)[MAXR], const float (&prv)[MAXR]) {
  float q = 0.f;
#pragma unroll
  for (int t = 0; t < MAXR; ++t) {
    if (t < a.r) {
      const float x = plu[t] + prv[t] - __ldg(a.mu + k * a.r + t);
      const float s = __ldg(a.sinv + k * a.r + t);
      q = fmaf(x * x, s * s, q);
    }
  }
  return __expf(-0.5f * q);
}

__device__ __forceinline__ void load_p(const float* p, int r, float (&x)[MAXR]) {
#pragma unroll
  for (int t = 0; t < MAXR; ++t) x[t] = t < r ? __ldg(p + t) : 0.f;
}

// Lane groups for the column passes (K8 forward, pass 2): L lanes own one row and a warp walks
// 32 / L rows, L = 8 / 16 / 32 for K f <= 64 / 128 / 256 (each lane keeps 8 accumulators, columns
// sl, sl + L, ...).  On Pubmed-shaped layers (4.5 edges per row, K f = 48) a whole warp per row left
// most lanes idle in the per-edge weight stage and most of the warp's latency uncovered.
template <int L>
struct alignas(16) GmmGroupSmem {
  uint32_t nb[L];
  float w[L * (MAXK + 1)];
  float red[8 * L];
  float row[8 * L];
};

template <int L>
struct GmmGroup {
  int sub, sl;
  unsigned mask;
  __device__ __forceinline__ GmmGroup() {
    const int lane = threadIdx.x & 31;
    sub = lane / L;
    sl = lane % L;
    mask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (sub * L));
  }
  __device__ __forceinline__ int slot() const { return (threadIdx.x >> 5) * (32 / L) + sub; }
  __device__ __forceinline__ int64_t row() const { return ((int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5)) * (32 / L) + sub; }
  __device__ __forceinline__ float sum(float v) const {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
    return v;
  }
};

template <int L>
__global__ void __launch_bounds__(256, GNNCG_GMM_MINB_FWD) gmm_fwd_kernel(GmmArgs a) {
  constexpr int NA = 8;  // accumulators per lane: K f <= 8 L
  __shared__ GmmGroupSmem<L> smem[WARPS * (32 / L)];
  const GmmGroup<L> grp;
  GmmGroupSmem<L>& sm = smem[grp.slot()];
  const int64_t v = grp.row();
  if (v >= a.rows) return;
  const int K = a.K, r = a.r, f = a.f, Kf = K * f;
  float prv[MAXR];
  load_p(a.Y + v * a.ldy + Kf + r, r, prv);
  float acc[NA];
#pragma unroll
  for (int i = 0; i < NA; ++i) acc[i] = 0.f;
  const uint64_t e0 = a.off[v], e1 = a.off[v + 1];
  for (uint64_t base = e0; base < e1; base += L) {
    const int n = (int)min((uint64_t)L, e1 - base);
    if (grp.sl < n) {
      const uint32_t u = __ldg(a.nbr + base + grp.sl);
      sm.nb[grp.sl] = u;
      float plu[MAXR];
      load_p(a.Y + (int64_t)u * a.ldy + Kf, r, plu);
#pragma unroll
      for (int k = 0; k < MAXK; ++k)
        if (k < K) sm.w[grp.sl * (MAXK + 1) + k] = gmm_w(a, k, plu, prv);
    }
    __syncwarp(grp.mask);
    for (int j = 0; j < n; ++j) {
      const float* y = a.Y + (int64_t)sm.nb[j] * a.ldy;
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        const int c = i * L + grp.sl;
        if (c < Kf) acc[i] = fmaf(sm.w[j * (MAXK + 1) + c / f], __ldg(y + c), acc[i]);
      }
    }
    __syncwarp(grp.mask);
  }
#pragma unroll
  for (int i = 0; i < NA; ++i) {
    const int c = i * L + grp.sl;
    if (c < Kf) sm.red[c] = acc[i];
  }
  __syncwarp(grp.mask);
  const float invK = 1.f / (float)K;
  for (int c = grp.sl; c < f; c += L) {
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += sm.red[k * f + c];
    a.out[v * f + c] = s * invK;
  }
}

// pass 1 over csr_dst, in lane groups (see gmm_fwd_kernel): lane per edge.  The per-row dmu / dsinv
// partials (2 K r <= 64 values) are reduced across the group per L-edge batch and accumulated in
// the group's shared-memory slot in batch order.
template <int L>
struct alignas(16) GmmDstSmem {
  float row[8 * L];
  float part[2 * MAXK * MAXR];
};

template <int L>
__global__ void __launch_bounds__(256, GNNCG_GMM_MINB) gmm_bwd_dst_kernel(GmmArgs a) {
  __shared__ GmmDstSmem<L> smem[WARPS * (32 / L)];
  const GmmGroup<L> grp;
  GmmDstSmem<L>& sm = smem[grp.slot()];
  const int64_t v = grp.row();
  if (v >= a.rows) return;
  const int K = a.K, r = a.r, f = a.f, Kf = K * f, Kr = K * r;
  const float invK = 1.f / (float)K;
  for (int c = grp.sl; c < f; c += L) sm.row[c] = __ldg(a.dOut + v * f + c);
  for (int c = grp.sl; c < 2 * Kr; c += L) sm.part[c] = 0.f;
  __syncwarp(grp.mask);
  float prv[MAXR], dpr[MAXR];
  load_p(a.Y + v * a.ldy + Kf + r, r, prv);
#pragma unroll
  for (int t = 0; t < MAXR; ++t) dpr[t] = 0.f;
  const uint64_t e0 = a.off[v], e1 = a.off[v + 1];
  for (uint64_t base = e0; base < e1; base += L) {
    const bool valid = base + grp.sl < e1;
    const int64_t u = valid ? (int64_t)__ldg(a.nbr + base + grp.sl) : 0;
    const float* y = a.Y + u * a.ldy;
    float plu[MAXR], dw[MAXK];
    load_p(y + Kf, r, plu);
#pragma unroll
    for (int k = 0; k < MAXK; ++k) dw[k] = 0.f;
    if (valid && a.vec4) {
      for (int c = 0; c < f; c += 4) {
        const float4 g = *reinterpret_cast<const float4*>(sm.row + c);
#pragma unroll
        for (int k = 0; k < MAXK; ++k)
          if (k < K) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(y + k * f + c));
            dw[k] = fmaf(g.w, x.w, fmaf(g.z, x.z, fmaf(g.y, x.y, fmaf(g.x, x.x, dw[k]))));
          }
      }
    } else if (valid) {
      for (int c = 0; c < f; ++c) {
        const float g = sm.row[c];
#pragma unroll
        for (int k = 0; k < MAXK; ++k)
          if (k < K) dw[k] = fmaf(g, __ldg(y + k * f + c), dw[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < MAXK; ++k) {
      if (k < K) {
        const float dq = valid ? -0.5f * gmm_w(a, k, plu, prv) * dw[k] * invK : 0.f;
#pragma unroll
        for (int t = 0; t < MAXR; ++t) {
          if (t < r) {
            const float s = __ldg(a.sinv + k * r + t), x = plu[t] + prv[t] - __ldg(a.mu + k * r + t);
            const float dmd = dq * 2.f * x * s * s;
            dpr[t] += dmd;
            const float gm = grp.sum(-dmd), gs = grp.sum(dq * 2.f * x * x * s);
            if (grp.sl == 0) {
              sm.part[k * r + t] += gm;
              sm.part[Kr + k * r + t] += gs;
            }
          }
        }
      }
    }
  }
  __syncwarp(grp.mask);
  float* part = a.part + v * (int64_t)(2 * Kr);
  for (int c = grp.sl; c < 2 * Kr; c += L) part[c] = sm.part[c];
#pragma unroll
  for (int t = 0; t < MAXR; ++t) {
    if (t < r) {
      const float s = grp.sum(dpr[t]);
      if (grp.sl == 0) a.dY[v * a.ldy + Kf + r + t] = s;
    }
  }
}

// pass 2 over csc_src, in lane groups (see gmm_fwd_kernel).
template <int L>
__global__ void __launch_bounds__(256, GNNCG_GMM_MINB) gmm_bwd_src_kernel(GmmArgs a) {
  constexpr int NA = 8;
  __shared__ GmmGroupSmem<L> smem[WARPS * (32 / L)];
  const GmmGroup<L> grp;
  GmmGroupSmem<L>& sm = smem[grp.slot()];
  const int64_t u = grp.row();
  if (u >= a.rows) return;
  const int K = a.K, r = a.r, f = a.f, Kf = K * f;
  const float invK = 1.f / (float)K;
  const float* yu = a.Y + u * a.ldy;
  for (int c = grp.sl; c < Kf; c += L) sm.row[c] = __ldg(yu + c);
  float plu[MAXR], dpl[MAXR];
  load_p(yu + Kf, r, plu);
#pragma unroll
  for (int t = 0; t < MAXR; ++t) dpl[t] = 0.f;
  __syncwarp(grp.mask);
  float acc[NA];
#pragma unroll
  for (int i = 0; i < NA; ++i) acc[i] = 0.f;
  const uint64_t e0 = a.off[u], e1 = a.off[u + 1];
  for (uint64_t base = e0; base < e1; base += L) {
    const int n = (int)min((uint64_t)L, e1 - base);
    if (grp.sl < n) {
      const int64_t v = __ldg(a.nbr + base + grp.sl);
      sm.nb[grp.sl] = (uint32_t)v;
      float prv[MAXR], dw[MAXK];
      load_p(a.Y + v * a.ldy + Kf + r, r, prv);
      const float* g = a.dOut + v * f;
#pragma unroll
      for (int k = 0; k < MAXK; ++k) dw[k] = 0.f;
      if (a.vec4) {
        for (int c = 0; c < f; c += 4) {
          const float4 gc = __ldg(reinterpret_cast<const float4*>(g + c));
#pragma unroll
          for (int k = 0; k < MAXK; ++k)
            if (k < K) {
              const float4 x = *reinterpret_cast<const float4*>(sm.row + k * f + c);
              dw[k] = fmaf(gc.w, x.w, fmaf(gc.z, x.z, fmaf(gc.y, x.y, fmaf(gc.x, x.x, dw[k]))));
            }
        }
      } else {
        for (int c = 0; c < f; ++c) {
          const float gc = __ldg(g + c);
#pragma unroll
          for (int k = 0; k < MAXK; ++k)
            if (k < K) dw[k] = fmaf(gc, sm.row[k * f + c], dw[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < MAXK; ++k) {
        if (k < K) {
          const float w = gmm_w(a, k, plu, prv);
          sm.w[grp.sl * (MAXK + 1) + k] = w * invK;
          const float dq = -0.5f * w * dw[k] * invK;
#pragma unroll
          for (int t = 0; t < MAXR; ++t)
            if (t < r) {
              const float s = __ldg(a.sinv + k * r + t), x = plu[t] + prv[t] - __ldg(a.mu + k * r + t);
              dpl[t] = fmaf(dq * 2.f * x, s * s, dpl[t]);
            }
        }
      }
    }
    __syncwarp(grp.mask);
    for (int j = 0; j < n; ++j) {
      const float* g = a.dOut + (int64_t)sm.nb[j] * f;
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        const int c = i * L + grp.sl;
        if (c < Kf) acc[i] = fmaf(sm.w[j * (MAXK + 1) + c / f], __ldg(g + c % f), acc[i]);
      }
    }
    __syncwarp(grp.mask);
  }
  float* dy = a.dY + u * a.ldy;
#pragma unroll
  for (int i = 0; i < NA; ++i) {
    const int c = i * L + grp.sl;
    if (c < Kf) dy[c] = acc[i];
  }
  // alignment columns past K f + 2 r (rows padded to 16 bytes for the TMA GEMM): zero, so
  // dWcat = H^T dY leaves the padding of [W | P_l | P_r] at zero
  for (int64_t c = Kf + 2 * r + grp.sl; c < a.ldy; c += L) dy[c] = 0.f;
#pragma unroll
  for (int t = 0; t < MAXR; ++t) {
    if (t < r) {
      const float s = grp.sum(dpl[t]);
      if (grp.sl == 0) dy[Kf + t] = s;
    }
  }
}

// Lanes per row for the grouped passes and their grid.
int gmm_lanes(int Kf) { return Kf <= 64 ? 8 : Kf <= 128 ? 16 : 32; }
unsigned gmm_grid(int64_t rows, int L) { return (unsigned)ceil_div(rows, (int64_t)WARPS * (32 / L)); }

// dmu / dsinv = sum over rows of the per-row partials, in a fixed order (deterministic):
// stage 1: block b sums rows [b R, (b+1) R) -- thread t owns parameter t % n and rows
// t / n, t / n + G, ... (G = 256 / n groups), so each sweep reads G whole contiguous rows;
// the groups are merged in shared memory in group order.  stage 2: one warp per parameter
// sums the block partials.
constexpr int RED_THREADS = 256, RED_BLOCKS = 592;

int red_blocks(int64_t rows) {
  const int64_t b = ceil_div(rows, (int64_t)64);
  return (int)(b < 1 ? 1 : b > RED_BLOCKS ? RED_BLOCKS : b);
}

__global__ void __launch_bounds__(RED_THREADS) gmm_param_partial_kernel(int64_t rows, int n,
                                                                       const float* __restrict__ part,
                                                                       float* __restrict__ blk) {
  __shared__ float sm[RED_THREADS];
  const int t = threadIdx.x, G = RED_THREADS / n, grp = t / n, q = t - grp * n;
  const int64_t per = ceil_div(rows, (int64_t)gridDim.x);
  const int64_t r0 = blockIdx.x * per, r1 = r0 + per < rows ? r0 + per : rows;
  float s = 0.f;
  if (grp < G)
    for (int64_t rr = r0 + grp; rr < r1; rr += G) s += __ldg(part + rr * n + q);
  sm[t] = s;
  __syncthreads();
  if (t < n) {
    float acc = 0.f;
    for (int k = 0; k < G; ++k) acc += sm[k * n + t];
    blk[(int64_t)blockIdx.x * n + t] = acc;
  }
}

__global__ void gmm_param_reduce_kernel(int nblk, int n, const float* __restrict__ blk, float* __restrict__ dmu,
                                        float* __restrict__ dsinv, int Kr) {
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= n) return;
  float s = 0.f;
  for (int b = lane; b < nblk; b += 32) s += blk[(int64_t)b * n + q];
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
  GmmArgs a{csr->num_rows, K, r, f, csr->off, csr->nbr, Y, ldy, mu, sinv, nullptr, out, nullptr, nullptr, false};
  const int L = gmm_lanes(K * f);
  cudaStream_t s = as_stream(stream);
  if (L == 8) gmm_fwd_kernel<8><<<gmm_grid(csr->num_rows, 8), 256, 0, s>>>(a);
  else if (L == 16) gmm_fwd_kernel<16><<<gmm_grid(csr->num_rows, 16), 256, 0, s>>>(a);
  else gmm_fwd_kernel<32><<<gmm_grid(csr->num_rows, 32), 256, 0, s>>>(a);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

size_t gnncg_gmm_bwd_workspace(const gnncg_index_t* csr, int K, int r) {
  if (!csr) return 0;
  const size_t n = (size_t)2 * K * r;
  return align_up((size_t)csr->num_rows * n * sizeof(float)) + align_up((size_t)red_blocks(csr->num_rows) * n * sizeof(float));
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
            static_cast<float*>(ws),
            f % 4 == 0 && ldy % 4 == 0 && (uintptr_t)Y % 16 == 0 && (uintptr_t)dOut % 16 == 0};
  const int L = gmm_lanes(K * f);
  if (L == 8) gmm_bwd_dst_kernel<8><<<gmm_grid(csr->num_rows, 8), 256, 0, s>>>(a);
  else if (L == 16) gmm_bwd_dst_kernel<16><<<gmm_grid(csr->num_rows, 16), 256, 0, s>>>(a);
  else gmm_bwd_dst_kernel<32><<<gmm_grid(csr->num_rows, 32), 256, 0, s>>>(a);
  GNNCG_LAUNCH_CHECK();
  a.off = csc->off;
  a.nbr = csc->nbr;
  if (L == 8) gmm_bwd_src_kernel<8><<<gmm_grid(csr->num_rows, 8), 256, 0, s>>>(a);
  else if (L == 16) gmm_bwd_src_kernel<16><<<gmm_grid(csr->num_rows, 16), 256, 0, s>>>(a);
  else gmm_bwd_src_kernel<32><<<gmm_grid(csr->num_rows, 32), 256, 0, s>>>(a);
  GNNCG_LAUNCH_CHECK();
  const int n = 2 * K * r, nblk = red_blocks(csr->num_rows);
  float* blk = a.part + align_up((size_t)csr->num_rows * n * sizeof(float)) / sizeof(float);
  gmm_param_partial_kernel<<<nblk, RED_THREADS, 0, s>>>(csr->num_rows, n, a.part, blk);
  GNNCG_LAUNCH_CHECK();
  gmm_param_reduce_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, s>>>(nblk, n, blk, dmu, dsinv, K * r);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

}  // extern "C"
