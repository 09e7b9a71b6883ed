// SPDX-License-Identifier: Apache-2.0
//
// Dense transforms on the 5th-gen tensor cores (K1 / K5 on sm_100a):
//   C[M,N] = op(A)[M,K] op(B)[K,N], fp32 in / fp32 out, fp32-accurate via a 3xTF32
//   split: x = hi + lo (hi = x with the low 13 mantissa bits cleared, lo = x - hi
//   exactly), C = A_hi B_hi + A_hi B_lo + A_lo B_hi accumulated in TMEM.  The tensor core
//   truncates fp32 operands to tf32, so the raw landed tile IS hi: only lo is materialised
//   (pinned by tests/test_gpu_gemm_tc.py::test_tc_gemm_identity_split).
// Replaces matmul / matmul_nt / matmul_tn (proj/src/tensor.cpp:8-60) for the
// reorganized ApplyVertex(W) of the GNN layers and its two backward Applies.
//
// Default kernel (gemm_tf32x3_persist_kernel): one CTA per SM walks the output tiles;
//   warp 0       TMA producer: cp.async.bulk.tensor 2D boxes of A and B
//   warp 1       TMEM allocator + single-thread tcgen05.mma issuer (kind::tf32)
//   warps 2..11  split warps: lo of each landed stage in shared memory
//   warps 12..15 epilogue: tcgen05.ld 32x32b.x32 from TMEM -> registers -> global
// mbarrier pipeline: full (TMA bytes) -> split -> MMA -> empty (tcgen05.commit); the
// accumulator is double-buffered in TMEM (accfull / accempty), so tile i's epilogue overlaps
// tile i+1's main loop.  gemm_tf32x3_kernel (GNNCG_TC_PERSIST=0) is the one-tile-per-CTA form.
// Operands may be K-major (SWIZZLE_64B rows of BK = 16 fp32) or MN-major (transposed;
// SWIZZLE_128B_BASE32B boxes of 32 elements x BK k-rows).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace gnncg_b200 {
namespace tc {

// BK fp32 = 64 B: K-major tiles are SWIZZLE_64B rows (8-row atoms 512 B apart); MN-major tiles
// are SWIZZLE_128B_BASE32B boxes of 32 elements x BK k-rows.  A 48 KB stage (128 x 256 tile:
// raw/hi + lo of A and B) gives a 4-deep pipeline in 192 KB.
constexpr int BM = 128, BK = 16;
constexpr int SPLIT_WARPS = 8;                     // split + epilogue warps (2 per TMEM lane quadrant)
constexpr int THREADS = 64 + 32 * SPLIT_WARPS;    // + TMA producer warp + MMA warp

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE_BYTES = 2 * (A_BYTES + B_BYTES);  // raw->hi and lo of A and B
  static constexpr int STAGES = (192 * 1024) / STAGE_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// SM100 shared-memory matrix descriptor, version 1.  layout: 4 = SWIZZLE_64B (K-major
// operands), 1 = SWIZZLE_128B_BASE32B (the only layout for MN-major 32-bit operands:
// Swizzle<2,5,2>, atoms of 32 elements x 4 k-rows).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                              uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  d |= (uint64_t)layout << 61;
  return d;
}

// Instruction descriptor: kind::tf32, fp32 accumulate, M = 128, N = BN.
__host__ __device__ constexpr uint32_t instr_desc(int N, bool a_mn, bool b_mn) {
  return (1u << 4)                   // c_format = F32
         | (2u << 7)                 // a_format = TF32
         | (2u << 10)                // b_format = TF32
         | ((a_mn ? 1u : 0u) << 15)  // a_major
         | ((b_mn ? 1u : 0u) << 16)  // b_major
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_c, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_c),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Load + wait in ONE asm statement: the destination registers are undefined until
// tcgen05.wait::ld, so the compiler must not see them as defined in between.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}

// lo = x - hi of a landed stage (hi = the raw tile itself: the tensor core truncates to tf32).
__device__ __forceinline__ void split_lo(const float* raw, float* lo, int bytes, int tid, int nthr) {
  const float4* r4 = reinterpret_cast<const float4*>(raw);
  float4* l4 = reinterpret_cast<float4*>(lo);
  const int n = bytes / 16;
  for (int i = tid; i < n; i += nthr) {
    const float4 v = r4[i];
    float4 h;
    h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
    h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
    h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
    h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
    l4[i] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
  }
}

// A_MN: A stored K x M (M contiguous); else M x K.  B_MN: B stored K x N (N contiguous); else N x K.
// epi.Al != null (K1 of the GAT layer, no split-K, f % 32 == 0, BN % f == 0): the epilogue also
// forms the reorganized attention LPs of every output row from the accumulator it already holds,
//   Al[row, k] = <C[row, k*f : (k+1)*f], a_l[k, :]>,  Ar likewise,
// in the same sequential order as gat.cu's attn_dots_kernel (bitwise identical results).
template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                       float* __restrict__ C, int64_t ldc, int64_t M, int64_t N, int64_t K, int64_t kchunk,
                       int64_t split_stride, int dbg, AttnEpi epi) {
  using CF = Cfg<BN>;
  constexpr int S = CF::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * CF::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* split = bars + S;
  uint64_t* empty = bars + 2 * S;
  uint64_t* accum = bars + 3 * S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;  // M tiles on x: no 65535 limit
  const int64_t kb0 = (int64_t)blockIdx.z * kchunk;
  const int64_t kb1 = min(K, kb0 + kchunk);
  const int nk = (int)((kb1 - kb0 + BK - 1) / BK);
  float* Cz = C + (int64_t)blockIdx.z * split_stride;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&split[s], 32 * SPLIT_WARPS);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a));
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b));
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  auto a_hi = [&](int s) { return reinterpret_cast<float*>(smem + s * CF::STAGE_BYTES); };
  auto a_lo = [&](int s) { return reinterpret_cast<float*>(smem + s * CF::STAGE_BYTES + CF::A_BYTES); };
  auto b_hi = [&](int s) { return reinterpret_cast<float*>(smem + s * CF::STAGE_BYTES + 2 * CF::A_BYTES); };
  auto b_lo = [&](int s) {
    return reinterpret_cast<float*>(smem + s * CF::STAGE_BYTES + 2 * CF::A_BYTES + CF::B_BYTES);
  };

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      for (int i = 0; i < nk; ++i) {
        const int s = i % S;
        const uint32_t ph = (uint32_t)(i / S) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_expect_tx(&full[s], CF::A_BYTES + CF::B_BYTES);
        const int k = (int)(kb0 + (int64_t)i * BK);
        if (!A_MN) {
          tma_load_2d(a_hi(s), &map_a, k, (int)m0, &full[s]);
        } else {
#pragma unroll
          for (int j = 0; j < BM / 32; ++j)
            tma_load_2d(reinterpret_cast<uint8_t*>(a_hi(s)) + j * (32 * BK * 4), &map_a, (int)m0 + 32 * j, k,
                        &full[s]);
        }
        if (!B_MN) {
          tma_load_2d(b_hi(s), &map_b, k, (int)n0, &full[s]);
        } else {
#pragma unroll
          for (int j = 0; j < BN / 32; ++j)
            tma_load_2d(reinterpret_cast<uint8_t*>(b_hi(s)) + j * (32 * BK * 4), &map_b, (int)n0 + 32 * j, k,
                        &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      constexpr uint32_t idesc = instr_desc(BN, A_MN, B_MN);
      // K-major (SW64): rows of 64 B, 8-row atoms 512 B apart (SBO), k-step = +32 B.
      // MN-major (SW128_32B): 32-element x BK-k boxes (32 BK 4 B) along MN (LBO), 4-k-row
      // atoms 512 B apart (SBO), k-step (8 rows) = +1024 B.
      constexpr uint32_t MNBOX = 32 * BK * 4;
      const uint32_t a_lbo = A_MN ? MNBOX : 16u, a_sbo = 512u, a_step = A_MN ? 1024u : 32u;
      const uint32_t b_lbo = B_MN ? MNBOX : 16u, b_sbo = 512u, b_step = B_MN ? 1024u : 32u;
      const uint32_t a_lay = A_MN ? 1u : 4u, b_lay = B_MN ? 1u : 4u;
      for (int i = 0; i < nk; ++i) {
        const int s = i % S;
        const uint32_t ph = (uint32_t)(i / S) & 1u;
        mbar_wait(&split[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t ah = smem_u32(a_hi(s)), al = smem_u32(a_lo(s));
        const uint32_t bh = smem_u32(b_hi(s)), bl = smem_u32(b_lo(s));
#pragma unroll
        for (int k = 0; k < BK / 8; ++k) {
          const uint64_t dah = smem_desc(ah + k * a_step, a_lbo, a_sbo, a_lay);
          const uint64_t dal = smem_desc(al + k * a_step, a_lbo, a_sbo, a_lay);
          const uint64_t dbh = smem_desc(bh + k * b_step, b_lbo, b_sbo, b_lay);
          const uint64_t dbl = smem_desc(bl + k * b_step, b_lbo, b_sbo, b_lay);
          mma_tf32(tmem, dah, dbh, idesc, (i > 0 || k > 0) ? 1u : 0u);
          mma_tf32(tmem, dah, dbl, idesc, 1u);
          mma_tf32(tmem, dal, dbh, idesc, 1u);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(accum);
    }
  } else {
    // ---- split warps (2..5), then epilogue
    const int tid = threadIdx.x - 64;
    for (int i = 0; i < nk; ++i) {
      const int s = i % S;
      const uint32_t ph = (uint32_t)(i / S) & 1u;
      mbar_wait(&full[s], ph);
      split_lo(a_hi(s), a_lo(s), CF::A_BYTES, tid, 32 * SPLIT_WARPS);
      split_lo(b_hi(s), b_lo(s), CF::B_BYTES, tid, 32 * SPLIT_WARPS);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&split[s]);
    }
    const int q = warp & 3;  // TMEM lane quadrant of this warp (hardware: warp w reads lanes 32 (w % 4) ..)
    // the two warps of a quadrant take the first / second half of the column chunks
    const int half = (warp - 2) / 4;
    constexpr int NCH = BN / 32 / (SPLIT_WARPS / 4);
    const int64_t row = m0 + q * 32 + lane;
    if (nk > 0) {
      mbar_wait(accum, 0);
      asm volatile("tcgen05.fence::after_thread_sync;");
    }
    float dl = 0.f, dr = 0.f;  // attention-LP partial sums of the current head (epi.Al)
#pragma unroll 1
    for (int c = half * NCH; c < (half + 1) * NCH; ++c) {
      uint32_t r[32];
      if (dbg == 1) {  // debug: bypass TMEM, write a coordinate pattern
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = __float_as_uint((float)(row * 1000 + c * 32 + j));
      } else if (dbg == 2) {  // debug: first raw smem words of stage 0 (A hi)
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = reinterpret_cast<const uint32_t*>(smem)[(lane * 32 + j) & 4095];
      } else if (nk > 0) {
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 32), r);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = 0u;
      }
      const int64_t col = n0 + c * 32;
      if (row < M) {
        float* dst = Cz + row * ldc + col;
        if (col + 32 <= N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(dst + j) = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                              __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col + j < N) dst[j] = __uint_as_float(r[j]);
        }
      }
      if (epi.Al != nullptr && col < N) {  // whole chunk inside one head (f % 32 == 0)
        const float* pl = epi.a_l + col;
        const float* pr = epi.a_r + col;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float x = __uint_as_float(r[j]);
          dl = fmaf(x, __ldg(pl + j), dl);
          dr = fmaf(x, __ldg(pr + j), dr);
        }
        if ((col + 32) % epi.f == 0) {
          if (row < M) {
            const int64_t k = (col + 32) / epi.f - 1;
            epi.Al[row * epi.h + k] = dl;
            epi.Ar[row * epi.h + k] = dr;
          }
          dl = dr = 0.f;
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
  }
}

// ------------------------------------------------------------------------ persistent variant
// One CTA per SM walks the output tiles (M fastest, then N, then the split-K slice).  The stage
// ring runs continuously across tiles, and the accumulator is double-buffered in TMEM
// (2 x BN columns), so the epilogue of tile i (its own 4 warps, one per TMEM lane quadrant)
// overlaps the TMA / split / MMA work of tile i+1, and no CTA pays the TMEM allocation and
// pipeline fill per tile.
//   warp 0 TMA producer | warp 1 MMA issuer | warps 2..11 split | warps 12..15 epilogue
// Split warps (lo = x - tf32(x) of each landed stage): 10 measured best where both operands are
// split per stage (dW = H^T dHt: C2 0.337 vs 0.373 ms, C5 5.18 vs 6.19 ms); the GEMMs whose B
// (the weight) is pre-split are unchanged (profiles/r02_gemm_split.txt).  P_EPI_WARP0 must stay
// a multiple of 4 (the epilogue warps' TMEM lane quadrants): 2, 6, 10, ...
#ifndef GNNCG_TC_SPLIT_WARPS
#define GNNCG_TC_SPLIT_WARPS 10
#endif
constexpr int P_SPLIT_WARPS = GNNCG_TC_SPLIT_WARPS;
constexpr int P_EPI_WARP0 = 2 + P_SPLIT_WARPS;  // 8: warp % 4 == TMEM lane quadrant
constexpr int P_THREADS = 32 * (P_EPI_WARP0 + 4);

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(P_THREADS, 1)
    gemm_tf32x3_persist_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                               const __grid_constant__ CUtensorMap map_blo, int b_presplit, float* __restrict__ C,
                               int64_t ldc, int64_t M, int64_t N, int64_t K, int64_t kchunk, int64_t split_stride,
                               int tiles_m, int tiles_n, int64_t tiles, AttnEpi epi) {
  static_assert(P_EPI_WARP0 % 4 == 0, "epilogue warps must start on a lane-quadrant boundary");
  using CF = Cfg<BN>;
  constexpr int S = CF::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * CF::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* split = bars + S;
  uint64_t* empty = bars + 2 * S;
  uint64_t* accfull = bars + 3 * S;       // [2]
  uint64_t* accempty = bars + 3 * S + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&split[s], 32 * P_SPLIT_WARPS);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a));
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b));
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  auto a_hi = [&](int s) { return reinterpret_cast<float*>(smem + s * CF::STAGE_BYTES); };
  auto a_lo = [&](int s) { return reinterpret_cast<float*>(smem + s * CF::STAGE_BYTES + CF::A_BYTES); };
  auto b_hi = [&](int s) { return reinterpret_cast<float*>(smem + s * CF::STAGE_BYTES + 2 * CF::A_BYTES); };
  auto b_lo = [&](int s) {
    return reinterpret_cast<float*>(smem + s * CF::STAGE_BYTES + 2 * CF::A_BYTES + CF::B_BYTES);
  };
  // tile t -> (m0, n0, k range, split slice)
  struct Tile {
    int64_t m0, n0, kb0;
    int nk, z;
  };
  auto tile_of = [&](int64_t t) {
    Tile x;
    const int64_t mt = t % tiles_m, rest = t / tiles_m;
    x.m0 = mt * BM;
    x.n0 = (rest % tiles_n) * BN;
    x.z = (int)(rest / tiles_n);
    x.kb0 = (int64_t)x.z * kchunk;
    const int64_t kb1 = min(K, x.kb0 + kchunk);
    x.nk = (int)((kb1 - x.kb0 + BK - 1) / BK);
    return x;
  };

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      uint32_t g = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const Tile x = tile_of(t);
        for (int i = 0; i < x.nk; ++i, ++g) {
          const int s = (int)(g % S);
          const uint32_t ph = (g / S) & 1u;
          mbar_wait(&empty[s], ph ^ 1u);
          mbar_expect_tx(&full[s], CF::A_BYTES + CF::B_BYTES * (b_presplit ? 2 : 1));
          const int k = (int)(x.kb0 + (int64_t)i * BK);
          if (b_presplit) {  // B's lo was materialised once in global memory (the reused weight)
            if (!B_MN) {
              tma_load_2d(b_lo(s), &map_blo, k, (int)x.n0, &full[s]);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 32; ++j)
                tma_load_2d(reinterpret_cast<uint8_t*>(b_lo(s)) + j * (32 * BK * 4), &map_blo, (int)x.n0 + 32 * j, k,
                            &full[s]);
            }
          }
          if (!A_MN) {
            tma_load_2d(a_hi(s), &map_a, k, (int)x.m0, &full[s]);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 32; ++j)
              tma_load_2d(reinterpret_cast<uint8_t*>(a_hi(s)) + j * (32 * BK * 4), &map_a, (int)x.m0 + 32 * j, k,
                          &full[s]);
          }
          if (!B_MN) {
            tma_load_2d(b_hi(s), &map_b, k, (int)x.n0, &full[s]);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 32; ++j)
              tma_load_2d(reinterpret_cast<uint8_t*>(b_hi(s)) + j * (32 * BK * 4), &map_b, (int)x.n0 + 32 * j, k,
                          &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      constexpr uint32_t idesc = instr_desc(BN, A_MN, B_MN);
      constexpr uint32_t MNBOX = 32 * BK * 4;
      const uint32_t a_lbo = A_MN ? MNBOX : 16u, a_sbo = 512u, a_step = A_MN ? 1024u : 32u;
      const uint32_t b_lbo = B_MN ? MNBOX : 16u, b_sbo = 512u, b_step = B_MN ? 1024u : 32u;
      const uint32_t a_lay = A_MN ? 1u : 4u, b_lay = B_MN ? 1u : 4u;
      uint32_t g = 0, it = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
        const Tile x = tile_of(t);
        const uint32_t b = it & 1u, use = it >> 1;
        mbar_wait(&accempty[b], (use & 1u) ^ 1u);  // the epilogue has drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d = tmem + b * BN;
        for (int i = 0; i < x.nk; ++i, ++g) {
          const int s = (int)(g % S);
          const uint32_t ph = (g / S) & 1u;
          mbar_wait(&split[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t ah = smem_u32(a_hi(s)), al = smem_u32(a_lo(s));
          const uint32_t bh = smem_u32(b_hi(s)), bl = smem_u32(b_lo(s));
#pragma unroll
          for (int k = 0; k < BK / 8; ++k) {
            const uint64_t dah = smem_desc(ah + k * a_step, a_lbo, a_sbo, a_lay);
            const uint64_t dal = smem_desc(al + k * a_step, a_lbo, a_sbo, a_lay);
            const uint64_t dbh = smem_desc(bh + k * b_step, b_lbo, b_sbo, b_lay);
            const uint64_t dbl = smem_desc(bl + k * b_step, b_lbo, b_sbo, b_lay);
            mma_tf32(d, dah, dbh, idesc, (i > 0 || k > 0) ? 1u : 0u);
            mma_tf32(d, dah, dbl, idesc, 1u);
            mma_tf32(d, dal, dbh, idesc, 1u);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&accfull[b]);
      }
    }
  } else if (warp < P_EPI_WARP0) {
    // ---- split warps: lo of every landed stage
    const int tid = threadIdx.x - 64;
    uint32_t g = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      const Tile x = tile_of(t);
      for (int i = 0; i < x.nk; ++i, ++g) {
        const int s = (int)(g % S);
        const uint32_t ph = (g / S) & 1u;
        mbar_wait(&full[s], ph);
        split_lo(a_hi(s), a_lo(s), CF::A_BYTES, tid, 32 * P_SPLIT_WARPS);
        if (!b_presplit) split_lo(b_hi(s), b_lo(s), CF::B_BYTES, tid, 32 * P_SPLIT_WARPS);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&split[s]);
      }
    }
  } else {
    // ---- epilogue warps: TMEM -> registers -> global (+ the attention LPs)
    const int q = warp & 3;
    uint32_t it = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const Tile x = tile_of(t);
      const uint32_t b = it & 1u, use = it >> 1;
      mbar_wait(&accfull[b], use & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;");
      float* Cz = C + (int64_t)x.z * split_stride;
      const int64_t row = x.m0 + q * 32 + lane;
      float dl = 0.f, dr = 0.f;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + b * BN + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 32), r);
        const int64_t col = x.n0 + c * 32;
        if (row < M) {
          float* dst = Cz + row * ldc + col;
          if (col + 32 <= N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *reinterpret_cast<float4*>(dst + j) = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                                __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col + j < N) dst[j] = __uint_as_float(r[j]);
          }
        }
        if (epi.Al != nullptr && col < N) {  // whole chunk inside one head (f % 32 == 0)
          const float* pl = epi.a_l + col;
          const float* pr = epi.a_r + col;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float xv = __uint_as_float(r[j]);
            dl = fmaf(xv, __ldg(pl + j), dl);
            dr = fmaf(xv, __ldg(pr + j), dr);
          }
          if ((col + 32) % epi.f == 0) {
            if (row < M) {
              const int64_t k = (col + 32) / epi.f - 1;
              epi.Al[row * epi.h + k] = dl;
              epi.Ar[row * epi.h + k] = dr;
            }
            dl = dr = 0.f;
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(&accempty[b]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
  }
}

// ---------------------------------------------------------------------------------- host
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D fp32 tensor map: inner dim `inner` (contiguous), outer dim `outer`, row stride `ld` elements.
bool make_map(CUtensorMap* map, const float* ptr, int64_t inner, int64_t outer, int64_t ld, int box_inner,
              int box_outer, bool mn_major) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// GNNCG_TC_PERSIST=0 selects the one-tile-per-CTA kernel.
bool persist_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("GNNCG_TC_PERSIST");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <int BN, bool A_MN, bool B_MN>
int launch(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int64_t M, int64_t N,
           int64_t K, int splits, int64_t kchunk, int64_t split_stride, cudaStream_t s, const AttnEpi& epi,
           const float* B_lo, int64_t ldb_lo) {
  using CF = Cfg<BN>;
  CUtensorMap ma, mb, mbl;
  bool ok = A_MN ? make_map(&ma, A, M, K, lda, 32, BK, true) : make_map(&ma, A, K, M, lda, BK, BM, false);
  ok = ok && (B_MN ? make_map(&mb, B, N, K, ldb, 32, BK, true) : make_map(&mb, B, K, N, ldb, BK, BN, false));
  const bool presplit = B_lo != nullptr && persist_enabled();
  mbl = mb;
  if (presplit)
    ok = ok && (B_MN ? make_map(&mbl, B_lo, N, K, ldb_lo, 32, BK, true)
                     : make_map(&mbl, B_lo, K, N, ldb_lo, BK, BN, false));
  if (!ok) return fail(GNNCG_ERR_CUDA, "gemm_tc: cuTensorMapEncodeTiled failed");
  if (persist_enabled()) {
    auto pk = gemm_tf32x3_persist_kernel<BN, A_MN, B_MN>;
    static bool pattr = false;
    if (!pattr) {
      GNNCG_CUDA_TRY(cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));
      pattr = true;
    }
    const int tm = (int)ceil_div(M, BM), tn = (int)ceil_div(N, BN);
    const int64_t tiles = (int64_t)tm * tn * splits;
    static int sms = 0;
    if (sms == 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    }
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, sms);
    pk<<<grid, P_THREADS, CF::SMEM, s>>>(ma, mb, mbl, presplit ? 1 : 0, C, ldc, M, N, K, kchunk, split_stride, tm, tn,
                                         tiles, epi);
    GNNCG_LAUNCH_CHECK();
    return GNNCG_OK;
  }
  auto kern = gemm_tf32x3_kernel<BN, A_MN, B_MN>;
  static bool attr_set = false;
  if (!attr_set) {
    GNNCG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));
    attr_set = true;
  }
  dim3 grid((unsigned)ceil_div(M, BM), (unsigned)ceil_div(N, BN), (unsigned)splits);
  static int dbg = -1;
  if (dbg < 0) {
    const char* e = getenv("GNNCG_TC_DEBUG");
    dbg = e ? atoi(e) : 0;
  }
  kern<<<grid, THREADS, CF::SMEM, s>>>(ma, mb, C, ldc, M, N, K, kchunk, split_stride, dbg, epi);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

}  // namespace tc

// N-tile width: 256 for wide outputs, or 128 when GNNCG_TC_BN=128 (a 3-stage pipeline instead
// of 2 stages of the 96 KB 128x256 tile).
int tc_bn(int64_t N) {
  static int force = -1;
  if (force < 0) {
    const char* e = getenv("GNNCG_TC_BN");
    force = e ? atoi(e) : 0;
  }
  if (force == 128) return 128;
  return N > 128 ? 256 : 128;
}

// Entry used by gnncg_gemm (gemm.cu).  trans_a: A stored K x M ; trans_b: B stored N x K.
// In the tensor-core kernel's terms A is MN-major iff trans_a, B is MN-major iff !trans_b.
bool tc_gemm_eligible(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                      const float* B, int64_t ldb) {
  if (!tc::encode_fn()) return false;
  if (M <= 0 || N <= 0 || K <= 0) return false;
  if (((uintptr_t)A & 15) || ((uintptr_t)B & 15) || (lda % 4) || (ldb % 4)) return false;
  if (M >= (1ll << 31) || N >= (1ll << 31) || K >= (1ll << 31)) return false;
  (void)trans_a;
  (void)trans_b;
  return true;
}

int tc_gemm(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
            int64_t ldb, float* C, int64_t ldc, int splits, int64_t kchunk, float* partial, cudaStream_t s,
            const AttnEpi& epi, const float* B_lo, int64_t ldb_lo) {
  float* out = splits > 1 ? partial : C;
  const int64_t ldo = splits > 1 ? N : ldc;
  const int64_t stride = splits > 1 ? M * N : 0;
  const bool a_mn = trans_a != 0, b_mn = trans_b == 0;
  const bool wide = tc_bn(N) == 256;
#define GNNCG_TC(BN, AM, BMN) \
  return tc::launch<BN, AM, BMN>(A, lda, B, ldb, out, ldo, M, N, K, splits, kchunk, stride, s, epi, B_lo, ldb_lo)
  if (wide) {
    if (!a_mn && !b_mn) GNNCG_TC(256, false, false);
    if (!a_mn && b_mn) GNNCG_TC(256, false, true);
    if (a_mn && !b_mn) GNNCG_TC(256, true, false);
    GNNCG_TC(256, true, true);
  } else {
    if (!a_mn && !b_mn) GNNCG_TC(128, false, false);
    if (!a_mn && b_mn) GNNCG_TC(128, false, true);
    if (a_mn && !b_mn) GNNCG_TC(128, true, false);
    GNNCG_TC(128, true, true);
  }
#undef GNNCG_TC
}

}  // namespace gnncg_b200
