// SPDX-License-Identifier: Apache-2.0
//
// Dense transforms (K1 / K5): ApplyVertex(W) and its two backward Applies.
// Replaces matmul / matmul_nt / matmul_tn (proj/src/tensor.cpp:8-60).
//
// fp32 in, fp32 accumulate (the reference computes these in T = float/double;
// SPEC.md:139).  This translation unit is the CUDA-core SIMT path: 128x128x16
// CTA tiles, 8x8 register micro-tiles, double-buffered shared memory, and a
// deterministic split-K (fixed-order partial reduction) for the tall-skinny
// Hᵀ·dH̃ weight gradient (K = |V|).  The GEMMs are <= ~6% of the GAT layer step
// (SURVEY §7 "Hard parts"), the fused gather kernels dominate.
#include "common.cuh"

namespace gnncg_b200 {
namespace {

constexpr int BM = 128, BN = 128, BK = 16, NT = 256;

template <bool TA, bool TB>
__global__ void __launch_bounds__(NT, 2)
    sgemm_kernel(int64_t M, int64_t N, int64_t K, const float* __restrict__ A, int64_t lda,
                 const float* __restrict__ B, int64_t ldb, float* __restrict__ C, int64_t ldc, int64_t kchunk,
                 int64_t split_stride) {
  __shared__ __align__(16) float As[2][BK][BM];
  __shared__ __align__(16) float Bs[2][BK][BN];
  const int t = threadIdx.x;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;  // M tiles on x: no 65535 limit
  const int64_t kb = (int64_t)blockIdx.z * kchunk;
  const int64_t ke = min(K, kb + kchunk);
  float* Cz = C + (int64_t)blockIdx.z * split_stride;

  float ra[8], rb[8];
  auto load_tile = [&](int64_t k0) {
    if (!TA) {  // A[m*lda + k]
      const int ml = t >> 1, kl = (t & 1) * 8;
      const int64_t m = m0 + ml;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t k = k0 + kl + i;
        ra[i] = (m < M && k < ke) ? __ldg(A + m * lda + k) : 0.f;
      }
    } else {  // A[k*lda + m]
      const int kl = t >> 4, ml = (t & 15) * 8;
      const int64_t k = k0 + kl;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t m = m0 + ml + i;
        ra[i] = (m < M && k < ke) ? __ldg(A + k * lda + m) : 0.f;
      }
    }
    if (!TB) {  // B[k*ldb + n]
      const int kl = t >> 4, nl = (t & 15) * 8;
      const int64_t k = k0 + kl;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t n = n0 + nl + i;
        rb[i] = (n < N && k < ke) ? __ldg(B + k * ldb + n) : 0.f;
      }
    } else {  // B[n*ldb + k]
      const int nl = t >> 1, kl = (t & 1) * 8;
      const int64_t n = n0 + nl;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t k = k0 + kl + i;
        rb[i] = (n < N && k < ke) ? __ldg(B + n * ldb + k) : 0.f;
      }
    }
  };
  auto store_tile = [&](int buf) {
    if (!TA) {
      const int ml = t >> 1, kl = (t & 1) * 8;
#pragma unroll
      for (int i = 0; i < 8; ++i) As[buf][kl + i][ml] = ra[i];
    } else {
      const int kl = t >> 4, ml = (t & 15) * 8;
      *reinterpret_cast<float4*>(&As[buf][kl][ml]) = make_float4(ra[0], ra[1], ra[2], ra[3]);
      *reinterpret_cast<float4*>(&As[buf][kl][ml + 4]) = make_float4(ra[4], ra[5], ra[6], ra[7]);
    }
    if (!TB) {
      const int kl = t >> 4, nl = (t & 15) * 8;
      *reinterpret_cast<float4*>(&Bs[buf][kl][nl]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
      *reinterpret_cast<float4*>(&Bs[buf][kl][nl + 4]) = make_float4(rb[4], rb[5], rb[6], rb[7]);
    } else {
      const int nl = t >> 1, kl = (t & 1) * 8;
#pragma unroll
      for (int i = 0; i < 8; ++i) Bs[buf][kl + i][nl] = rb[i];
    }
  };

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  const int tx = t & 15, ty = t >> 4;
  int buf = 0;
  if (kb < ke) {
    load_tile(kb);
    store_tile(0);
    __syncthreads();
  }
  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
    const bool more = k0 + BK < ke;
    if (more) load_tile(k0 + BK);
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][k][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (more) {
      store_tile(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (n < N) Cz[m * ldc + n] = acc[i][j];
    }
  }
}

// C[m,n] = sum_z P[z][m][n] (deterministic split-K merge).
#ifndef GNNCG_SPLITK_WARPS
#define GNNCG_SPLITK_WARPS 8
#endif
// Split-K partials summed in a fixed order.  A block takes 32 outputs at a time; warp w adds splits
// w, w + 8, ... (one coalesced 128-byte row per split) and the 8 warp sums are added in warp order.
// (One thread per output walking all splits left each thread a chain of up to 64 loads: 14-16 us
// per launch for the 8K-output weight gradients of EdgeConv / MoNet.)
__global__ void __launch_bounds__(32 * GNNCG_SPLITK_WARPS) splitk_reduce_kernel(int64_t M, int64_t N, int splits,
                                                                              const float* __restrict__ P,
                                                                              float* __restrict__ C, int64_t ldc) {
  constexpr int W = GNNCG_SPLITK_WARPS;
  __shared__ float red[W][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t total = M * N;
  for (int64_t i0 = (int64_t)blockIdx.x * 32; i0 < total; i0 += (int64_t)gridDim.x * 32) {
    const int64_t i = i0 + lane;
    float s = 0.f;
    if (i < total) {
#pragma unroll 4
      for (int z = w; z < splits; z += W) s += P[(int64_t)z * total + i];
    }
    red[w][lane] = s;
    __syncthreads();
    if (w == 0 && i < total) {
      float t = red[0][lane];
#pragma unroll
      for (int k = 1; k < W; ++k) t += red[k][lane];
      C[(i / N) * ldc + (i % N)] = t;
    }
    __syncthreads();
  }
}
unsigned splitk_grid(int64_t total) { return (unsigned)std::min<int64_t>(ceil_div(total, (int64_t)32), 148 * 8); }

int choose_splits(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ceil_div(M, BM) * ceil_div(N, BN);
  if (tiles >= 2 * 148 || K < 4 * 256) return 1;
  int64_t s = ceil_div(2 * 148, tiles);
  s = std::min<int64_t>(s, K / 256);
  s = std::min<int64_t>(s, 64);
  return (int)std::max<int64_t>(s, 1);
}

}  // namespace

// Tensor-core path (gemm_tc.cu).
int tc_bn(int64_t N);
bool tc_gemm_eligible(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                      const float* B, int64_t ldb);
int tc_gemm(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
            int64_t ldb, float* C, int64_t ldc, int splits, int64_t kchunk, float* partial, cudaStream_t s,
            const AttnEpi& epi, const float* B_lo = nullptr, int64_t ldb_lo = 0);

namespace {
// GNNCG_GEMM=simt forces the CUDA-core kernel (A/B comparisons); default: tensor cores when eligible.
bool tc_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("GNNCG_GEMM");
    v = (e && strcmp(e, "simt") == 0) ? 0 : 1;
  }
  return v == 1;
}

// The reused operand of a tall GEMM (the weight: B of H W and of dHt W^T) is split into its
// tf32 lo part once per call into the workspace, so the kernel's split warps only process A.
// presplit_b_bytes: the bytes of that dense copy ((rows, cols) = B as stored), or 0 when unused.

__global__ void presplit_lo_kernel(int64_t rows, int64_t cols, const float* __restrict__ B, int64_t ldb,
                                   float* __restrict__ lo) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    const float x = __ldg(B + r * ldb + c);
    lo[i] = x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  }
}

int tc_splits(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ceil_div(M, 128) * ceil_div(N, tc_bn(N));
  if (tiles >= 148 || K < 1024) return 1;
  // floor: tiles * splits <= 148, one tile per SM of the persistent kernel (a 150th tile would
  // double the kernel time); slices of >= 256 k (16 stages)
  int64_t s = std::min<int64_t>(148 / tiles, K / 256);
  return (int)std::max<int64_t>(std::min<int64_t>(s, 64), 1);
}
size_t presplit_b_bytes(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K) {
  const int64_t rows = trans_b ? N : K, cols = trans_b ? K : N;
  if (trans_a || cols % 4 != 0 || M < 16384 || rows * cols > (4 << 20) || tc_splits(M, N, K) != 1) return 0;
  return align_up((size_t)rows * cols * sizeof(float));
}
}  // namespace
}  // namespace gnncg_b200

using namespace gnncg_b200;

extern "C" {

size_t gnncg_gemm_workspace(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K) {
  const int s = std::max(choose_splits(M, N, K), tc_splits(M, N, K));
  const size_t split = s > 1 ? align_up((size_t)s * M * N * sizeof(float)) : 0;
  return std::max(split, presplit_b_bytes(trans_a, trans_b, M, N, K));
}

int gnncg_gemm(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
               const float* B, int64_t ldb, float* C, int64_t ldc, void* ws, size_t ws_bytes, void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(M >= 0 && N >= 0 && K >= 0, GNNCG_ERR_SHAPE, "gemm: negative dimension");
  GNNCG_REQUIRE(!(trans_a && trans_b), GNNCG_ERR_UNSUPPORTED, "gemm: A^T B^T not supported");
  GNNCG_REQUIRE(ldc >= N, GNNCG_ERR_SHAPE, "gemm: ldc < N");
  if (M == 0 || N == 0) return GNNCG_OK;
  if (K == 0) {  // empty contraction: C = 0
    GNNCG_REQUIRE(C, GNNCG_ERR_ARG, "gemm: null C");
    GNNCG_CUDA_TRY(cudaMemset2DAsync(C, ldc * sizeof(float), 0, N * sizeof(float), M, as_stream(stream)));
    return GNNCG_OK;
  }
  GNNCG_REQUIRE(lda >= (trans_a ? M : K) && ldb >= (trans_b ? K : N), GNNCG_ERR_SHAPE,
                "gemm: leading dimension too small");
  GNNCG_REQUIRE(A && B && C, GNNCG_ERR_ARG, "gemm: null pointer");
  cudaStream_t s = as_stream(stream);
  const size_t need = gnncg_gemm_workspace(trans_a, trans_b, M, N, K);
  GNNCG_REQUIRE(ws_bytes >= need && (need == 0 || ws), GNNCG_ERR_WORKSPACE, "gemm: workspace %zu < %zu", ws_bytes,
                need);
  if (tc_enabled() && tc_gemm_eligible(trans_a, trans_b, M, N, K, A, lda, B, ldb)) {
    int splits = tc_splits(M, N, K);
    const int64_t kchunk = splits > 1 ? ceil_div(ceil_div(K, splits), 32) * 32 : K;
    splits = splits > 1 ? (int)ceil_div(K, kchunk) : 1;  // every split gets >= 1 k-block
    const float* B_lo = nullptr;
    int64_t ldb_lo = 0;
    if (splits == 1 && presplit_b_bytes(trans_a, trans_b, M, N, K) > 0) {
      const int64_t rows = trans_b ? N : K, cols = trans_b ? K : N;
      presplit_lo_kernel<<<(unsigned)std::min<int64_t>(ceil_div(rows * cols, 256), 148 * 8), 256, 0, s>>>(
          rows, cols, B, ldb, static_cast<float*>(ws));
      GNNCG_LAUNCH_CHECK();
      B_lo = static_cast<const float*>(ws);
      ldb_lo = cols;
    }
    int rc = tc_gemm(trans_a, trans_b, M, N, K, A, lda, B, ldb, C, ldc, splits, kchunk, static_cast<float*>(ws), s,
                     AttnEpi{}, B_lo, ldb_lo);
    if (rc != GNNCG_OK) return rc;
    if (splits > 1) {
      splitk_reduce_kernel<<<splitk_grid(M * N), 32 * GNNCG_SPLITK_WARPS, 0, s>>>(M, N, splits, static_cast<float*>(ws),
                                                                                C, ldc);
      GNNCG_LAUNCH_CHECK();
    }
    return GNNCG_OK;
  }
  const int splits = choose_splits(M, N, K);
  const int64_t kchunk = splits > 1 ? ceil_div(ceil_div(K, splits), BK) * BK : std::max<int64_t>(K, 1);
  const int real_splits = splits > 1 ? (int)ceil_div(K, kchunk) : 1;
  dim3 grid((unsigned)ceil_div(M, BM), (unsigned)ceil_div(N, BN), (unsigned)real_splits);
  float* out = splits > 1 ? static_cast<float*>(ws) : C;
  const int64_t ldo = splits > 1 ? N : ldc;
  const int64_t stride = splits > 1 ? M * N : 0;
  if (!trans_a && !trans_b)
    sgemm_kernel<false, false><<<grid, NT, 0, s>>>(M, N, K, A, lda, B, ldb, out, ldo, kchunk, stride);
  else if (!trans_a && trans_b)
    sgemm_kernel<false, true><<<grid, NT, 0, s>>>(M, N, K, A, lda, B, ldb, out, ldo, kchunk, stride);
  else
    sgemm_kernel<true, false><<<grid, NT, 0, s>>>(M, N, K, A, lda, B, ldb, out, ldo, kchunk, stride);
  GNNCG_LAUNCH_CHECK();
  if (splits > 1) {
    splitk_reduce_kernel<<<splitk_grid(M * N), 32 * GNNCG_SPLITK_WARPS, 0, s>>>(M, N, real_splits, out, C, ldc);
    GNNCG_LAUNCH_CHECK();
  }
  return GNNCG_OK;
}

int gnncg_gat_transform(int64_t M, int64_t K, int heads, int f, const float* H, int64_t ldh, const float* W,
                        float* Ht, const float* a_l, const float* a_r, float* Al, float* Ar, void* ws,
                        size_t ws_bytes, void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(M >= 0 && K >= 0 && heads >= 1 && f >= 1, GNNCG_ERR_SHAPE, "gat_transform: bad shape");
  const int64_t N = (int64_t)heads * f;
  if (M == 0) return GNNCG_OK;
  GNNCG_REQUIRE(H && W && Ht && a_l && a_r && Al && Ar, GNNCG_ERR_ARG, "gat_transform: null pointer");
  GNNCG_REQUIRE(ldh >= K, GNNCG_ERR_SHAPE, "gat_transform: ldh < K");
  cudaStream_t s = as_stream(stream);
  const int bn = tc_bn(N);
  // (a head's column chunks must stay within one epilogue warp's half of the tile)
  if (K > 0 && tc_enabled() && tc_splits(M, N, K) == 1 && f % 32 == 0 && (bn / 2) % f == 0 &&
      tc_gemm_eligible(0, 0, M, N, K, H, ldh, W, N)) {
    AttnEpi epi;
    epi.a_l = a_l; epi.a_r = a_r; epi.Al = Al; epi.Ar = Ar; epi.h = heads; epi.f = f;
    const float* W_lo = nullptr;
    if (presplit_b_bytes(0, 0, M, N, K) > 0) {
      GNNCG_REQUIRE(ws && ws_bytes >= presplit_b_bytes(0, 0, M, N, K), GNNCG_ERR_WORKSPACE,
                    "gat_transform: workspace too small");
      presplit_lo_kernel<<<(unsigned)std::min<int64_t>(ceil_div(K * N, 256), 148 * 8), 256, 0, s>>>(
          K, N, W, N, static_cast<float*>(ws));
      GNNCG_LAUNCH_CHECK();
      W_lo = static_cast<const float*>(ws);
    }
    cost_add(kCostLp, (uint64_t)M, 1, s);  // the epilogue forms A_l / A_r of all M rows
    return tc_gemm(0, 0, M, N, K, H, ldh, W, N, Ht, N, 1, K, nullptr, s, epi, W_lo, N);
  }
  // unfused: the GEMM, then the LP kernel
  int rc = gnncg_gemm(0, 0, M, N, K, H, ldh, W, N, Ht, N, ws, ws_bytes, stream);
  if (rc != GNNCG_OK) return rc;
  return gnncg_gat_attn_dots(M, heads, f, Ht, a_l, a_r, Al, Ar, stream);
}

}  // extern "C"
