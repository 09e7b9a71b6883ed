// SPDX-License-Identifier: Apache-2.0
//
// TMA-fed variants of the fused GAT region kernels (K2 forward, fused fast K4).
//
// Same math and work items as gat.cu (see there for the semantics and citations);
// what changes is how neighbour feature rows reach the SM.  In gat.cu every lane
// issues 16-byte loads into registers, so the bytes in flight per SM are bounded by
// the register file (U rows x 1 KB per warp).  Here one lane per row issues a TMA
// bulk copy (cp.async.bulk global -> shared, completion counted in bytes on an
// mbarrier) of the whole row into a per-warp shared-memory ring of G groups x R rows;
// the warp consumes group g (LDS.128 + FMA) while groups g+1 .. g+G-1 are in flight,
// and refills the slot with group g+G as soon as it is drained.  Warps are persistent
// and pull work items from an atomic counter (results do not depend on the order).
#include <cfloat>

#include "common.cuh"
#include "gat_common.cuh"

namespace gnncg_b200 {
namespace gat {
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
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
__device__ __forceinline__ void bulk_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

constexpr int TW = 8;  // warps per CTA (persistent, one CTA per SM)

struct FwdWarp {
  uint32_t nb[32];
  float t0[32 * TS];
  float stat[4][MAXH];
  uint64_t full[16];
  int item;
};

// Ring geometry for a row of `rb` bytes: R rows per group (R | 32), G groups.
struct Ring {
  int R, G;
  __host__ __device__ static Ring make(int rb) {
    Ring r;
    r.R = rb <= 1024 ? 8 : (rb <= 2048 ? 4 : 2);
    r.G = 3;
    return r;
  }
  __host__ __device__ int bytes(int rb) const { return R * G * rb; }
};

// Issue the row copies of group `g` (edges [e0 + g*R, ...) of the item) into ring slot g % G.
__device__ __forceinline__ void issue_group(int lane, int64_t g, uint64_t e0, uint64_t e1, const uint32_t* __restrict__ nbr,
                                            const float* __restrict__ rows, int hf, uint8_t* ring, const Ring& rg,
                                            uint64_t* full, int64_t gc_base) {
  const uint64_t ge = e0 + (uint64_t)g * rg.R;
  if (ge >= e1) return;
  const int n = (int)min((uint64_t)rg.R, e1 - ge);
  const int slot = (int)((gc_base + g) % rg.G);
  const uint32_t rb = (uint32_t)hf * 4u;
  if (lane == 0) mbar_expect_tx(&full[slot], (uint32_t)n * rb);
  __syncwarp();
  if (lane < n) {
    const uint32_t u = __ldg(nbr + ge + lane);
    bulk_row(ring + ((size_t)slot * rg.R + lane) * rb, rows + (int64_t)u * hf, rb, &full[slot]);
  }
}

// ---------------------------------------------------------------------------
// K2 forward, TMA-fed.  VW = 4 (16-byte columns), any NV.
// ---------------------------------------------------------------------------
template <int NV>
__global__ void __launch_bounds__(TW * 32, 1) gat_fwd_tma_kernel(GatParams p, int* __restrict__ counter) {
  extern __shared__ __align__(128) uint8_t dsm[];
  constexpr int VW = 4;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int h = p.h, f = p.f, hf = h * f;
  const int rb = hf * 4;
  const Ring rg = Ring::make(rb);
  FwdWarp& sm = reinterpret_cast<FwdWarp*>(dsm)[w];
  uint8_t* ring = dsm + TW * sizeof(FwdWarp) + (size_t)w * rg.bytes(rb);
  if (lane < rg.G) mbar_init(&sm.full[lane], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const float slope = p.slope;
  const Cols<VW, NV> cols(lane, hf, f);
  int64_t gc = 0;  // groups issued so far by this warp (ring position / mbarrier phase)

  for (;;) {
    if (lane == 0) sm.item = atomicAdd(counter, 1);
    __syncwarp();
    const int64_t wi = sm.item;
    __syncwarp();
    if (wi >= p.num_items) break;
    const Item it = decode_item(p.items, p.off, wi, p.num_split_items, p.chunk);
    const uint64_t e0 = it.e0, e1 = it.e1;
    const int64_t ngroups = (int64_t)((e1 - e0 + rg.R - 1) / rg.R);
    for (int64_t g = 0; g < rg.G && g < ngroups; ++g) issue_group(lane, g, e0, e1, p.nbr, p.Ht, hf, ring, rg, sm.full, gc);

    if (lane < h) sm.stat[3][lane] = __ldg(p.Ar + (int64_t)it.row * h + lane);
    float M[MAXH], Sl[MAXH];
#pragma unroll
    for (int k = 0; k < MAXH; ++k) { M[k] = -FLT_MAX; Sl[k] = 0.f; }
    Vec<VW> acc[NV];
    zero(acc);
    __syncwarp();

    int64_t g = 0;
    for (uint64_t base = e0; base < e1; base += 32) {
      const int n = (int)min((uint64_t)32, e1 - base);
      const bool valid = lane < n;
      const uint32_t u = valid ? __ldg(p.nbr + base + lane) : 0u;
      float al[MAXH];
      load_heads(p.Al + (int64_t)u * h, h, al);
#pragma unroll
      for (int k = 0; k < MAXH; ++k) {
        if (k < h) {
          const float s = valid ? lrelu(al[k] + sm.stat[3][k], slope) : -FLT_MAX;
          const float mnew = fmaxf(M[k], warp_max(s));
          const float sc = __expf(M[k] - mnew);
          const float pk = valid ? __expf(s - mnew) : 0.f;
          M[k] = mnew;
          Sl[k] = fmaf(Sl[k], sc, pk);
          sm.t0[lane * TS + k] = pk;
          if (lane == 0) sm.stat[2][k] = sc;
        }
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const float sc = sm.stat[2][cols.hd[i]];
#pragma unroll
        for (int q = 0; q < VW; ++q) acc[i].x[q] *= sc;
      }
      // consume the block's groups
      for (int j0 = 0; j0 < n; j0 += rg.R, ++g) {
        const int slot = (int)((gc + g) % rg.G);
        mbar_wait(&sm.full[slot], (uint32_t)(((gc + g) / rg.G) & 1));
        const int nr = min(rg.R, n - j0);
        const uint8_t* sl = ring + (size_t)slot * rg.R * rb;
        for (int r = 0; r < nr; ++r) {
          const float* row = reinterpret_cast<const float*>(sl + (size_t)r * rb);
#pragma unroll
          for (int i = 0; i < NV; ++i) {
            if (cols.ok[i]) {
              const float4 x = *reinterpret_cast<const float4*>(row + cols.col[i]);
              const float a = sm.t0[(j0 + r) * TS + cols.hd[i]];
              acc[i].x[0] = fmaf(a, x.x, acc[i].x[0]);
              acc[i].x[1] = fmaf(a, x.y, acc[i].x[1]);
              acc[i].x[2] = fmaf(a, x.z, acc[i].x[2]);
              acc[i].x[3] = fmaf(a, x.w, acc[i].x[3]);
            }
          }
        }
        __syncwarp();  // slot drained by every lane
        if (g + rg.G < ngroups) issue_group(lane, g + rg.G, e0, e1, p.nbr, p.Ht, hf, ring, rg, sm.full, gc);
      }
    }
    gc += ngroups;

    const bool empty = e0 == e1;
#pragma unroll
    for (int k = 0; k < MAXH; ++k) {
      if (k < h) {
        const float S = warp_sum(Sl[k]);
        if (lane == 0) { sm.stat[0][k] = empty ? 0.f : M[k]; sm.stat[1][k] = S; }
      }
    }
    __syncwarp();
    if (!it.split) {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        if (cols.ok[i]) {
          const float den = sm.stat[1][cols.hd[i]];
          const float inv = den > 0.f ? 1.f / den : 0.f;
          Vec<VW> o;
#pragma unroll
          for (int q = 0; q < VW; ++q) o.x[q] = acc[i].x[q] * inv;
          st_vec<VW>(p.out + (int64_t)it.row * hf + cols.col[i], o);
        }
      }
      if (lane < h) {
        p.mo[(int64_t)it.row * h + lane] = sm.stat[0][lane];
        p.dd[(int64_t)it.row * h + lane] = sm.stat[1][lane];
      }
    } else {
      float* part = p.part + wi * fwd_stride(h, f);
#pragma unroll
      for (int i = 0; i < NV; ++i)
        if (cols.ok[i]) st_vec<VW>(part + cols.col[i], acc[i]);
      if (lane < h) {
        part[hf + lane] = sm.stat[0][lane];
        part[hf + h + lane] = sm.stat[1][lane];
      }
    }
    __syncwarp();
  }
}

}  // namespace

bool tma_fwd_supported(int h, int f) { return f % 4 == 0 && h * f <= 1024 && h * f >= 32; }

size_t tma_smem_bytes(int h, int f) {
  const int rb = h * f * 4;
  return TW * sizeof(FwdWarp) + (size_t)TW * Ring::make(rb).bytes(rb);
}

int launch_fwd_tma(const GatParams& p, int* counter, cudaStream_t s) {
  const int hf = p.h * p.f;
  const int nvec = (int)ceil_div(hf / 4, 32);
  const size_t smem = tma_smem_bytes(p.h, p.f);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  GNNCG_CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(int), s));
#define GNNCG_TMA_FWD(NV_)                                                                                   \
  do {                                                                                                       \
    GNNCG_CUDA_TRY(cudaFuncSetAttribute(gat_fwd_tma_kernel<NV_>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                        (int)smem));                                                         \
    gat_fwd_tma_kernel<NV_><<<sms, TW * 32, smem, s>>>(p, counter);                                          \
  } while (0)
  if (nvec <= 1) GNNCG_TMA_FWD(1);
  else if (nvec <= 2) GNNCG_TMA_FWD(2);
  else if (nvec <= 4) GNNCG_TMA_FWD(4);
  else GNNCG_TMA_FWD(8);
#undef GNNCG_TMA_FWD
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

}  // namespace gat
}  // namespace gnncg_b200
