// SPDX-License-Identifier: Apache-2.0
//
// K4f, wavefront-lean: the fused fast-mode GAT region backward over csc_src
// (gnncg_gat_bwd_src_fused) for row shapes that fill the warp exactly
// (h*f = 32*NV*VW, f/VW lanes per head, NV in {1, 2}: the Reddit shape 8 x 32 and
// the C5 shape 8 x 16).
//
// Same arithmetic as gat_bwd_src_fast_kernel (gat.cu): per out-edge e = (u -> v) of
// source u, alpha_e = exp(LReLU(A_l[u] + A_r[v]) - lse[v]), dalpha_e = <dOut[v], Ht[u]>
// per head, dz_e = LReLU'(z) alpha_e (dalpha_e - c[v]);  dHt[u] = sum alpha dOut[v]
// (+ LP terms), dA_l[u] = sum dz, dA_r[v] += dz (global reduction)
// (PAPER.md:615-662 ).
//
// Why a second kernel: ncu on B200 (profiles/r01_v12_ncu_full.json) shows the previous one
// bound by the L1 data pipe (l1tex__data_pipe_lsu_wavefronts 82% of peak), not by
// DRAM (54%) or L2 (52%).  22 wavefronts per edge: 15.4 global (8 of them the gathered
// 1 KB row, 6 the per-lane 96-byte destination records: 32 scattered 16-byte loads per
// instruction cost 32 wavefronts) and 6.6 shared (one LDS per gathered row for its id,
// one per row and vector for its weight).  This kernel keeps the row gather and cuts
// the rest:
//   * records are {A_r, lse, c, 0} per head (rec_stride = 4h): one 16-byte load per
//     (edge, head) pair, lanes = pairs, so an instruction reads 32/h whole 128-byte
//     records (4 wavefronts instead of 32), and each lane evaluates its own pair;
//   * the softmax weights are stored R = 4/NV rows x NV heads per 16 bytes in the
//     order the column mapping reads them: one broadcast LDS.128 per R rows;
//   * the gathered rows' ids are read four at a time (LDS.128 broadcast);
//   * (gate * alpha, c) per (edge, head) sit side by side: the dz stage reads one
//     8-byte pair per output.
// Lane layout at the Reddit shape (8 x 32): each lane owns 8 consecutive columns of ONE head
// (VW = 8, NV = 1, 4 lanes per head) and gathers them with one 256-bit load (LDG.E.ENL2.256):
// half the load instructions of the paired 2 x 128-bit layout (VW = 4, NV = 2, 8 lanes per
// head), and the per-edge head dots reduce over 4 lanes instead of 8 (6 shuffles and 12
// selects per 8-row group instead of 14 and 28).  Measured (same box, 3 rounds): K4f 9.9-10.0
// vs 10.6-10.7 ms, step 37.5-37.6 vs 38.8-39.3 ms; K2 unchanged (7.50-7.57 vs 7.57-7.65).
// The paired layout remains the path for tables that are only 16-byte aligned.
#include <algorithm>
#include <cstdint>
#include <cfloat>

#include "common.cuh"
#include "gat_common.cuh"

namespace gnncg_b200 {
namespace gat {
namespace {

template <int CNT, int OFF>
__device__ __forceinline__ void bfly(float* v, int lane) {
  if constexpr (OFF >= 1) {
    const bool up = (lane & OFF) != 0;
#pragma unroll
    for (int j = 0; j < CNT / 2; ++j) {
      const float send = up ? v[j] : v[j + CNT / 2];
      const float keep = up ? v[j + CNT / 2] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, OFF);
    }
    bfly<CNT / 2, OFF / 2>(v, lane);
  }
}

struct LeanSmem {
  uint32_t nb[kWarp];          // destination ids of the current 32-edge block
  float w[kWarp * MAXH];       // alpha, packed R rows x NV heads per float4
  float2 tc[kWarp * MAXH];     // (LReLU'(z) alpha, c) per (edge, head), tcidx order
  float dl[MAXH];              // dA_l[u] per head (item end)
};

// index of alpha(e, k) in LeanSmem::w: rows grouped by R = 4 / NV, heads by NV
template <int NV, int h>
__device__ __forceinline__ int widx(int e, int k) {
  constexpr int R = 4 / NV;
  return ((e / R) * (h / NV) + k / NV) * 4 + (e % R) * NV + (k % NV);
}

// index of (gate * alpha, c)(e, k) in LeanSmem::tc, laid out so that the two outputs of a
// lane in the dz stage are one 16-byte read: NV = 2 -> heads (2g, 2g+1) of one edge are
// adjacent; NV = 1 -> edges (2r, 2r+1) of one head are adjacent.  The 16-byte chunks are
// XOR-swizzled so that both the dz stage's reads (a quarter warp: 8 edges x one head pair, or
// 4 edge pairs x 2 heads) and the edge phase's 8-byte writes (a half warp: 2 edges x 8 heads)
// hit 8 distinct bank groups.  Unswizzled, the reads were 16-way conflicts: 16 wavefronts per
// 8-row group instead of 4 (ncu source page, profiles/r02_k4f_smem.md), 12 of K4f's ~55
// shared-pipe wavefronts per group.  h = 8 (lean kernels).
template <int NV, int h>
__device__ __forceinline__ int tcidx(int e, int k) {
  static_assert(h == 8, "tc swizzle: 8 heads");
  if constexpr (NV == 2) return (e * 4 + ((k >> 1) ^ ((e >> 1) & 3))) * 2 + (k & 1);
  else return ((e >> 1) * h + (k ^ (2 * ((e >> 1) & 3)))) * 2 + (e & 1);
}

__device__ __forceinline__ uint4 lds_u4(const uint32_t* p) { return *reinterpret_cast<const uint4*>(p); }

// Streaming accesses (read / written once per launch: the neighbour ids, the output rows) are
// marked evict-first so they do not displace the gathered rows in L2.  Measured (same box):
// C5 K2 73.4 vs 75.3 ms; C2 within noise (38.1-38.8 vs 38.3-38.7 ms per step).
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) { return __ldcs(p); }
template <int VW>
__device__ __forceinline__ void st_stream(float* p, const Vec<VW>& v) {
  static_assert(VW == 4 || VW == 8, "streaming store: 16- or 32-byte vectors");
  __stcs(reinterpret_cast<float4*>(p), make_float4(v.x[0], v.x[1], v.x[2], v.x[3]));
  if constexpr (VW == 8) __stcs(reinterpret_cast<float4*>(p) + 1, make_float4(v.x[4], v.x[5], v.x[6], v.x[7]));
}

// One gathered lane vector: VW = 8 is a single 256-bit load (LDG.E.ENL2.256, sm_100; the
// address is 32-byte aligned: 1 KB rows, 8-float lane columns), VW = 4 a 128-bit one.
template <int VW>
__device__ __forceinline__ Vec<VW> ldg_row(const float* p) {
  if constexpr (VW == 8) {
    Vec<8> r;
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]), "=f"(r.x[5]), "=f"(r.x[6]),
          "=f"(r.x[7])
        : "l"(p));
    return r;
  } else {
    return ldg_vec<VW>(p);
  }
}

// One lane vector of the bf16 gather table (the bf16 mode): VW bf16 = 8 or 16 bytes, kept packed.
template <int VW>
__device__ __forceinline__ Row<VW, true> ldg_row_lp(const char* p) {
  Row<VW, true> r;
  if constexpr (VW == 8) {
    const uint4 t = __ldg(reinterpret_cast<const uint4*>(p));
    r.w[0] = t.x; r.w[1] = t.y; r.w[2] = t.z; r.w[3] = t.w;
  } else {
    static_assert(VW == 4, "lean bf16 rows: 4 or 8 columns per lane");
    const uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
    r.w[0] = t.x; r.w[1] = t.y;
  }
  return r;
}

// gather_row (gat_common.cuh) with ldg_row: row r of a [*, hf] table at this lane's columns,
// fp32 (LP = false) or bf16 (LP = true, the bf16 mode's gather table).
template <int VW, int NV, bool LP>
__device__ __forceinline__ void lean_gather(const void* __restrict__ base, uint32_t r, int hf,
                                            const Cols<VW, NV>& c, Row<VW, LP> (&x)[NV]) {
  if constexpr (LP) {
    const uint64_t off = (uint64_t)r * (uint32_t)(hf * 2);
#pragma unroll
    for (int i = 0; i < NV; ++i)
      x[i] = ldg_row_lp<VW>(reinterpret_cast<const char*>(static_cast<const uint16_t*>(base) + c.col[i]) + off);
  } else {
    const uint64_t off = (uint64_t)r * (uint32_t)(hf * 4);
#pragma unroll
    for (int i = 0; i < NV; ++i)
      x[i].v = ldg_row<VW>(
          reinterpret_cast<const float*>(reinterpret_cast<const char*>(static_cast<const float*>(base) + c.col[i]) + off));
  }
}

// K2's row gathers of a [*, 8 F] table at this lane's paired columns (Cols with pl = F / VW:
// vector i sits F floats after vector i - 1).  The lane's base + column pointer is formed once
// and made opaque, so each row costs a 64-bit row * row_bytes + pointer (LEA + LEA.HI.X) and NV
// loads with immediate offsets; the plain (base + column) + row * row_bytes form compiles to 3
// IMADs and a MOV per row (the uniform table base folded into every address and the column
// re-added).  Measured at C2: K2 7.84 -> 7.62 ms; the same change made K4f slower (10.9 ->
// 11.4 ms: its loads issue later in the schedule), so K4f keeps gather_row.
template <int VW, int NV, int F, bool LP = false>
struct LaneRows {
  static constexpr uint32_t EB = LP ? 2u : 4u;  // bytes per element of the table
  const char* lb;
  __device__ __forceinline__ LaneRows(const void* base, int col0) {
    const void* b;
    if constexpr (LP) b = static_cast<const uint16_t*>(base) + col0;
    else b = static_cast<const float*>(base) + col0;
    asm("mov.b64 %0, %1;" : "=l"(lb) : "l"(b));
  }
  __device__ __forceinline__ void gather(uint32_t r, Row<VW, LP> (&x)[NV]) const {
    const char* a = lb + (uint64_t)r * (8u * F * EB);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      if constexpr (LP) x[i] = ldg_row_lp<VW>(a + i * F * EB);
      else x[i].v = ldg_row<VW>(reinterpret_cast<const float*>(a + i * F * EB));
    }
  }
};

template <int H, int VW, int NV, int PER, int WPC, int MINB, bool DYN, bool LP = false>
__global__ void __launch_bounds__(WPC * kWarp, MINB) gat_bwd_src_lean_kernel(GatParams p) {
  constexpr int U = 8;  // rows in flight per warp
  constexpr int R = 4 / NV;
  constexpr int NVAL = U * NV, NOUT = NVAL / PER;
  constexpr bool PAIR = NV == 2;  // lane's vectors in heads (2g, 2g+1): one 16-byte dA_r reduction per edge
  static_assert(NV == 1 || NV == 2, "lean K4f: one or two vectors per lane");
  static_assert(NVAL % PER == 0 && (!PAIR || NOUT == 2), "lean K4f: outputs per lane");
  __shared__ __align__(16) LeanSmem smem[WPC];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  LeanSmem& sm = smem[w];
  constexpr int h = H;  // compile-time heads: the edge phase's pair indexing is shifts, not divides
  const int f = p.f, hf = h * f;
  const float slope = p.slope;
  const int r = lane & (PER - 1);  // rank inside the head's lane group
  // column mapping: PAIR -> lane owns the same VW columns of heads 2 (lane / PER) + i;
  // NV = 1 -> columns lane * VW (head lane / PER)
  const Cols<VW, NV> cols(lane, hf, f, PAIR ? PER : 0);
  const int hd0 = cols.hd[0];
  constexpr int epi = kWarp / h;  // edges per edge-phase instruction
  const int kk = lane % h;        // edge phase: this lane's head
  unsigned nx = DYN && lane == 0 ? atomicAdd(p.ctr, (unsigned)p.batch) : 0u;
  int64_t cur = 0, cend = 0;
  for (int64_t g = blockIdx.x; DYN || g * WPC < p.num_items; g += gridDim.x) {
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
      wi = g * WPC + w;
      if (wi >= p.num_items) continue;
    }
    const Item it = decode_item(p.items, p.off, wi, p.num_split_items, p.chunk);
    count_item(p, it, lane);
    const int64_t u = it.row;
    const float alu = __ldg(p.Al + u * h + kk);
    Row<VW, LP> x[NV];  // the own row, as the forward aggregated it (bf16 mode: the bf16 Ht)
    Vec<VW> acc[NV];
    if constexpr (LP) {
      lean_gather<VW, NV, true>(p.lp_x, (uint32_t)u, hf, cols, x);
    } else {
      Vec<VW> xv[NV];
      gather_row<VW, NV>(p.Ht, (uint32_t)u, hf, cols, xv);
#pragma unroll
      for (int i = 0; i < NV; ++i) x[i].v = xv[i];
    }
    zero(acc);
    float dal[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) dal[i] = 0.f;

    const uint64_t e0 = it.e0, e1 = it.e1;
    uint32_t v_cur = e0 + lane < e1 ? ld_stream(p.nbr + e0 + lane) : 0u;
    const void* tab = LP ? static_cast<const void*>(p.lp) : static_cast<const void*>(p.dOut);
    for (uint64_t base = e0; base < e1; base += 32) {
      const int n = (int)min((uint64_t)32, e1 - base);
      sm.nb[lane] = v_cur;  // idle lanes hold row 0: a valid row whose weights are 0
      __syncwarp();
      Row<VW, LP> gv[U][NV];
      {  // the first half of the first row group goes out before the record loads
        const uint4 id4 = lds_u4(sm.nb);
        lean_gather<VW, NV, LP>(tab, id4.x, hf, cols, gv[0]);
        lean_gather<VW, NV, LP>(tab, id4.y, hf, cols, gv[1]);
        lean_gather<VW, NV, LP>(tab, id4.z, hf, cols, gv[2]);
        lean_gather<VW, NV, LP>(tab, id4.w, hf, cols, gv[3]);
      }
      {
        // edge phase, lanes = (edge, head) pairs: one {A_r, lse, c, 0} record load each
        float4 q[MAXH];
#pragma unroll
        for (int i = 0; i < MAXH; ++i) {
          if (i < h) {
            const int e = i * epi + lane / h;
            q[i] = __ldg(reinterpret_cast<const float4*>(p.rec + (int64_t)sm.nb[e] * (4 * h)) + kk);
          }
        }
#pragma unroll
        for (int i = 0; i < MAXH; ++i) {
          if (i < h) {
            const int e = i * epi + lane / h;
            const float z = alu + q[i].x;
            const float a = e < n ? __expf(lrelu(z, slope) - q[i].y) : 0.f;
            sm.w[widx<NV, h>(e, kk)] = a;
            sm.tc[tcidx<NV, h>(e, kk)] = make_float2(lrelu_grad(z, slope) * a, q[i].z);
          }
        }
      }
      __syncwarp();
      v_cur = base + 32 + lane < e1 ? ld_stream(p.nbr + base + 32 + lane) : 0u;
      {
        const uint4 id4 = lds_u4(sm.nb + 4);
        lean_gather<VW, NV, LP>(tab, id4.x, hf, cols, gv[4]);
        lean_gather<VW, NV, LP>(tab, id4.y, hf, cols, gv[5]);
        lean_gather<VW, NV, LP>(tab, id4.z, hf, cols, gv[6]);
        lean_gather<VW, NV, LP>(tab, id4.w, hf, cols, gv[7]);
      }
      for (int j = 0;;) {
        float pd[NVAL];
#pragma unroll
        for (int t = 0; t < U; t += R) {
          const float4 wv = *reinterpret_cast<const float4*>(sm.w + (((j + t) / R) * (h / NV) + hd0 / NV) * 4);
          const float wa[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
          for (int rr = 0; rr < R; ++rr)
#pragma unroll
            for (int i = 0; i < NV; ++i) {
              axpy_vec<VW>(wa[rr * NV + i], gv[t + rr][i], acc[i].x);
              pd[(t + rr) * NV + i] = dot_vec<VW>(x[i], gv[t + rr][i]);
            }
        }
        bfly<NVAL, PER / 2>(pd, lane);
        float dzp[NOUT];
        static_assert(NOUT == 2, "lean K4f: two dz outputs per lane (one 16-byte tc read)");
        // outputs q = 0, 1: NV = 2 -> edge j + r, heads hd0 + q; NV = 1 -> edge j + 2r + q, head hd0
        const float4 tc4 = *reinterpret_cast<const float4*>(sm.tc + tcidx<NV, h>(j + r * NOUT / NV, hd0));
#pragma unroll
        for (int q = 0; q < NOUT; ++q) {
          const int idx = r * NOUT + q;
          const int t = idx / NV, i = idx % NV;
          const int e = j + t;
          const int hd = hd0 + i;
          const float2 tc = q == 0 ? make_float2(tc4.x, tc4.y) : make_float2(tc4.z, tc4.w);
          const float dz = e < n ? tc.x * (pd[q] - tc.y) : 0.f;
#pragma unroll
          for (int ii = 0; ii < NV; ++ii)
            if (i == ii) dal[ii] += dz;
          dzp[q] = dz;
          // NV = 1: one 4-byte reduction per (edge, head).  Pairing heads into 8- / 16-byte
          // reductions through shuffles measured slower (C2 K4f 10.1 / 10.4 vs 10.0 ms)
          if (!PAIR && e < n) atomicAdd(p.dAro + (int64_t)sm.nb[e] * h + hd, dz);
        }

        if constexpr (PAIR) {
          // outputs (edge j + r, heads hd0, hd0 + 1); the next two heads of the same edge
          // are PER lanes up: even lane groups add four adjacent heads at once
          const float o0 = __shfl_down_sync(0xffffffffu, dzp[0], PER);
          const float o1 = __shfl_down_sync(0xffffffffu, dzp[1], PER);
          const int e = j + r;
          if (((lane / PER) & 1) == 0 && e < n)
            red_add_v4(p.dAro + (int64_t)sm.nb[e] * h + hd0, make_float4(dzp[0], dzp[1], o0, o1));
        }
        j += U;
        if (j >= n) break;
#pragma unroll
        for (int t = 0; t < U; t += 4) {
          const uint4 id4 = lds_u4(sm.nb + j + t);
          lean_gather<VW, NV, LP>(tab, id4.x, hf, cols, gv[t]);
          lean_gather<VW, NV, LP>(tab, id4.y, hf, cols, gv[t + 1]);
          lean_gather<VW, NV, LP>(tab, id4.z, hf, cols, gv[t + 2]);
          lean_gather<VW, NV, LP>(tab, id4.w, hf, cols, gv[t + 3]);
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
#pragma unroll
      for (int o = 1; o < PER; o <<= 1) dal[i] += __shfl_xor_sync(0xffffffffu, dal[i], o);
      if (r == 0) sm.dl[hd0 + i] = dal[i];
    }
    __syncwarp();
    if (!it.split) {
      if (lane < h) p.dAl[u * h + lane] = sm.dl[lane];
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const float dl = sm.dl[cols.hd[i]];
        const Vec<VW> al = ldg_vec<VW>(p.a_l + cols.col[i]);
        Vec<VW> o;
#pragma unroll
        for (int q = 0; q < VW; ++q) o.x[q] = fmaf(dl, al.x[q], acc[i].x[q]);
        st_stream<VW>(p.dHt + u * hf + cols.col[i], o);
      }
    } else {
      float* part = p.part + wi * src_stride(h, f);
#pragma unroll
      for (int i = 0; i < NV; ++i) st_vec<VW>(part + cols.col[i], acc[i]);
      if (lane < h) part[hf + lane] = sm.dl[lane];
    }
    __syncwarp();
  }  // work items
}

// ---------------------------------------------------------------------------
// K2, wavefront-lean: the fused forward region (Scatter(u_add_v) -> LeakyReLU ->
// edge-softmax -> Aggregate, RS1/RS2 PAPER.md:527-530) for the same
// shapes.  ncu on the previous kernel (gat_fwd_ovl_kernel): l1tex data pipe 90% of peak,
// half of it shared-memory wavefronts (8.3 per edge: an id LDS per gathered row, a weight
// LDS per row and vector, 4-way conflicting logit reads, per-lane exp-sum tables) plus
// 1.5 per edge of max-reduction shuffles.  Here the edge phase runs on (edge, head)
// pairs: each lane keeps one head, so the block max is a local max plus log2(32/h)
// shuffles, the exp-sum stays in a register, and the weights go to the packed table.
// ---------------------------------------------------------------------------
struct LeanFwdSmem {
  uint32_t nb[kWarp];     // source ids of the block (idle lanes: the last valid id)
  float w[kWarp * MAXH];  // exp(s - m), packed R rows x NV heads per float4
  float sc[MAXH];         // per head: rescale of the block, then 1 / exp-sum at the end
};

template <int H, int VW, int NV, int PER, int WPC, int MINB, bool DYN, bool LP = false>
__global__ void __launch_bounds__(WPC * kWarp, MINB) gat_fwd_lean_kernel(GatParams p) {
  constexpr int U = 8;
  constexpr int R = 4 / NV;
  __shared__ __align__(16) LeanFwdSmem smem[WPC];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  LeanFwdSmem& sm = smem[w];
  constexpr int h = H;  // compile-time heads: the edge phase's pair indexing is shifts, not divides
  const int f = p.f, hf = h * f;
  const float slope = p.slope;
  const Cols<VW, NV> cols(lane, hf, f, NV == 2 ? PER : 0);
  const int hd0 = cols.hd[0];
  constexpr int epi = kWarp / h;
  const int kk = lane % h;
  constexpr int F = PER * VW;  // = f: the shapes this kernel takes fill the warp
  const LaneRows<VW, NV, F, LP> hrows(LP ? static_cast<const void*>(p.lp) : static_cast<const void*>(p.Ht), cols.col[0]);
  unsigned nx = DYN && lane == 0 ? atomicAdd(p.ctr, 1u) : 0u;
  for (int64_t g = blockIdx.x; DYN || g * WPC < p.num_items; g += gridDim.x) {
    int64_t wi;
    if constexpr (DYN) {
      wi = __shfl_sync(0xffffffffu, nx, 0);
      if (wi >= p.num_items) break;
      if (lane == 0) nx = atomicAdd(p.ctr, 1u);
    } else {
      wi = g * WPC + w;
      if (wi >= p.num_items) continue;
    }
    const Item it = decode_item(p.items, p.off, wi, p.num_split_items, p.chunk);
    count_item(p, it, lane);
    const float arv = __ldg(p.Ar + (int64_t)it.row * h + kk);
    float m_run = -FLT_MAX, S = 0.f;  // this lane's head kk: running max, exp-sum partial
    Vec<VW> acc[NV];
    zero(acc);
    const uint64_t e0 = it.e0, e1 = it.e1;
    uint32_t u_cur = e0 + lane < e1 ? ld_stream(p.nbr + e0 + lane) : 0u;
    for (uint64_t base = e0; base < e1; base += 32) {
      const int n = (int)min((uint64_t)32, e1 - base);
      const uint32_t u_last = __shfl_sync(0xffffffffu, u_cur, n - 1);
      sm.nb[lane] = lane < n ? u_cur : u_last;  // rows past n repeat the last one (weight 0)
      __syncwarp();
      Row<VW, LP> x[U][NV];
#pragma unroll
      for (int t = 0; t < U; t += 4) {
        const uint4 id4 = lds_u4(sm.nb + t);
        hrows.gather(id4.x, x[t]);
        hrows.gather(id4.y, x[t + 1]);
        hrows.gather(id4.z, x[t + 2]);
        hrows.gather(id4.w, x[t + 3]);
      }
      // edge phase on (edge, head) pairs: logits of this lane's head for edges i*epi + lane/h
      float s[MAXH];
#pragma unroll
      for (int i = 0; i < MAXH; ++i)
        if (i < h) s[i] = __ldg(p.Al + (int64_t)sm.nb[i * epi + lane / h] * h + kk);
      u_cur = base + 32 + lane < e1 ? ld_stream(p.nbr + base + 32 + lane) : 0u;
      float mx = -FLT_MAX;
#pragma unroll
      for (int i = 0; i < MAXH; ++i) {
        if (i < h) {
          s[i] = i * epi + lane / h < n ? lrelu(s[i] + arv, slope) : -FLT_MAX;
          mx = fmaxf(mx, s[i]);
        }
      }
      for (int o = h; o < kWarp; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float m_new = fmaxf(m_run, mx);
      const float sc = __expf(m_run - m_new);
      float ps = 0.f;
#pragma unroll
      for (int i = 0; i < MAXH; ++i) {
        if (i < h) {
          const int e = i * epi + lane / h;
          const float pk = e < n ? __expf(s[i] - m_new) : 0.f;
          ps += pk;
          sm.w[widx<NV, h>(e, kk)] = pk;
        }
      }
      S = fmaf(S, sc, ps);
      m_run = m_new;
      if (lane < h) sm.sc[lane] = sc;
      __syncwarp();
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const float c = sm.sc[cols.hd[i]];
#pragma unroll
        for (int q = 0; q < VW; ++q) acc[i].x[q] *= c;
      }
      for (int j = 0;;) {
#pragma unroll
        for (int t = 0; t < U; t += R) {
          const float4 wv = *reinterpret_cast<const float4*>(sm.w + (((j + t) / R) * (h / NV) + hd0 / NV) * 4);
          const float wa[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
          for (int rr = 0; rr < R; ++rr)
#pragma unroll
            for (int i = 0; i < NV; ++i)
#pragma unroll
              for (int q = 0; q < VW; ++q) acc[i].x[q] = fmaf(wa[rr * NV + i], x[t + rr][i][q], acc[i].x[q]);
        }
        j += U;
        if (j >= n) break;
#pragma unroll
        for (int t = 0; t < U; t += 4) {
          const uint4 id4 = lds_u4(sm.nb + j + t);
          hrows.gather(id4.x, x[t]);
          hrows.gather(id4.y, x[t + 1]);
          hrows.gather(id4.z, x[t + 2]);
          hrows.gather(id4.w, x[t + 3]);
        }
      }
      __syncwarp();
    }
    for (int o = h; o < kWarp; o <<= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
    const float mk = e0 < e1 ? m_run : 0.f;
    if (!it.split) {
      if (lane < h) sm.sc[lane] = S > 0.f ? 1.f / S : 0.f;
      __syncwarp();
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const float inv = sm.sc[cols.hd[i]];
        Vec<VW> o;
#pragma unroll
        for (int q = 0; q < VW; ++q) o.x[q] = acc[i].x[q] * inv;
        st_stream<VW>(p.out + (int64_t)it.row * hf + cols.col[i], o);
      }
      if (lane < h) {
        p.mo[(int64_t)it.row * h + lane] = mk;
        p.dd[(int64_t)it.row * h + lane] = S;
      }
    } else {
      float* part = p.part + wi * fwd_stride(h, f);
#pragma unroll
      for (int i = 0; i < NV; ++i) st_vec<VW>(part + cols.col[i], acc[i]);
      if (lane < h) {
        part[hf + lane] = mk;
        part[hf + h + lane] = S;
      }
    }
    __syncwarp();
  }  // work items
}

// CTA shape of the lean kernels: warps per CTA and CTAs per SM (the launch bound caps the
// registers at 65536 / (MINB * WPC * 32)).  Overridable at build time for A/B runs.
// Measured on B200 (two boxes, ms per launch at C2, K4f / K2): 8 warps x 2 CTAs (128
// registers, 16 warps/SM) 11.49-11.62 / 7.94-8.03; 4 x 5 (96 registers, no spill, 20
// warps/SM) 10.78-10.92 / 7.71-7.81; 2 x 10 (96) 11.15-11.26 / 7.86-7.95; 2 x 12 (80, 24
// warps) 10.92-10.95 / 8.15-8.16; 2 x 16 (64, 32 warps) 11.95 / 7.68-7.75.  At C5: 4 x 5
// K4f 105.6 vs 113.0 ms, K2 82.5 vs 81.4 ms.  With the 256-bit lane rows (K4f needs fewer
// registers at 8 x 32) K4f moved to 4 x 7 (72 registers, 28 warps/SM): C2 9.23-9.35 vs 9.94-10.02
// ms (4 x 6: 9.47-9.54, 8 x 3: 9.46-9.52, 2 x 12: 9.45-9.57, 8 x 4: 9.64-9.70), C5 99.6 vs
// 100.6 ms (profiles/r02_cta.txt).  K2 at 8 x 32 (VW = 8) moved to 8 x 4 (64 registers, 32
// warps/SM): 7.53-7.58 vs 7.80 ms; at 8 x 16 (C5, VW = 4) it stays 4 x 5 (4 x 7
// there: 81.0 vs 75.6 ms).
#ifndef GNNCG_LEAN_FWD_WPC
#define GNNCG_LEAN_FWD_WPC 4
#endif
#ifndef GNNCG_LEAN_FWD_MINB
#define GNNCG_LEAN_FWD_MINB 5
#endif
#ifndef GNNCG_LEAN_FWD8_WPC
#define GNNCG_LEAN_FWD8_WPC 8
#endif
#ifndef GNNCG_LEAN_FWD8_MINB
#define GNNCG_LEAN_FWD8_MINB 4
#endif
#ifndef GNNCG_LEAN_BWD_WPC
#define GNNCG_LEAN_BWD_WPC 4
#endif
#ifndef GNNCG_LEAN_BWD_MINB
#define GNNCG_LEAN_BWD_MINB 7
#endif
// K2's shape per lane width: VW = 8 (8 x 32 rows) / VW = 4 (8 x 16 rows)
template <int VW>
struct FwdShape {
  static constexpr int WPC = VW == 8 ? GNNCG_LEAN_FWD8_WPC : GNNCG_LEAN_FWD_WPC;
  static constexpr int MINB = VW == 8 ? GNNCG_LEAN_FWD8_MINB : GNNCG_LEAN_FWD_MINB;
};
// K4f's shape: the one-head-per-lane layouts (NV = 1) at 4 x 7; the paired fallback (NV = 2,
// 16-byte aligned tables) keeps the 96-register 4 x 5 it was tuned at
template <int NV>
struct BwdShape {
  static constexpr int WPC = NV == 1 ? GNNCG_LEAN_BWD_WPC : 4;
  static constexpr int MINB = NV == 1 ? GNNCG_LEAN_BWD_MINB : 5;
};

int lean_num_sms() {
  static int v = 0;
  if (v == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
  }
  return v;
}

// persistent grid: MINB CTAs per SM, no more than the items need
unsigned lean_grid(int64_t items, int wpc, int minb) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(items, wpc), (int64_t)lean_num_sms() * minb));
}

// Launch with the L2 access-policy window of p.win (gnncg_l2_persist): the hottest rows of the
// gathered table are marked persisting, every other access streams.  Measured at C2 (same box,
// set-aside 30 / 60 MB vs off): K4f 10.56-10.76 vs 10.92-11.20 ms, K2 7.43-7.59 vs 7.67-7.87
// ms; 90+ MB slows the kernels between them (profiles/r02_l2_persist.txt).
template <typename... KArgs>
void launch_win(void (*k)(KArgs...), unsigned grid, unsigned block, cudaStream_t s, const GatParams& p) {
  if (p.win.bytes == 0) {
    k<<<grid, block, 0, s>>>(p);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeAccessPolicyWindow;
  at[0].val.accessPolicyWindow.base_ptr = const_cast<void*>(p.win.base);
  at[0].val.accessPolicyWindow.num_bytes = p.win.bytes;
  at[0].val.accessPolicyWindow.hitRatio = 1.0f;
  at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, p);
}

template <int VW, int NV, int PER>
void launch_fwd(const GatParams& p, cudaStream_t s) {
  constexpr int W = FwdShape<VW>::WPC, M = FwdShape<VW>::MINB;
  const unsigned grid = lean_grid(p.num_items, W, M);
  if (p.ctr) launch_win(gat_fwd_lean_kernel<8, VW, NV, PER, W, M, true>, grid, W * kWarp, s, p);
  else launch_win(gat_fwd_lean_kernel<8, VW, NV, PER, W, M, false>, grid, W * kWarp, s, p);
}

template <int VW, int NV, int PER>
void launch(const GatParams& p, cudaStream_t s) {
  constexpr int W = BwdShape<NV>::WPC, M = BwdShape<NV>::MINB;
  const unsigned grid = lean_grid(p.num_items, W, M);
  if (p.ctr) launch_win(gat_bwd_src_lean_kernel<8, VW, NV, PER, W, M, true>, grid, W * kWarp, s, p);
  else launch_win(gat_bwd_src_lean_kernel<8, VW, NV, PER, W, M, false>, grid, W * kWarp, s, p);
}

}  // namespace

// The shapes these kernels take: 8 heads, the row fills the warp (h f = 32 NV VW with VW = 4),
// one or two vectors per lane, f / 4 lanes per head dividing 32.
bool lean_supported(int h, int f) {
  // compiled for 8 heads: f = 32 (the Reddit shape, two vectors per lane in adjacent heads)
  // and f = 16 (the C5 shape, one vector per lane)
  return h == 8 && (f == 32 || f == 16);
}

bool lean_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("GNNCG_GAT_LEAN");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// The 256-bit lane rows need 32-byte aligned tables (rows are 1 KB): a caller's table that is
// only 16-byte aligned (a column view, an offset pointer) takes the paired 2 x 128-bit layout.
bool aligned32(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 31u) == 0; }

bool launch_fwd_lean(const GatParams& p, unsigned, cudaStream_t s) {
  if (!lean_enabled() || !lean_supported(p.h, p.f)) return false;
  if (p.f == 32) {
    if (aligned32(p.Ht)) launch_fwd<8, 1, 4>(p, s);
    else launch_fwd<4, 2, 8>(p, s);
  } else {
    launch_fwd<4, 1, 4>(p, s);
  }
  return true;
}

bool launch_bwd_src_lean(const GatParams& p, unsigned, cudaStream_t s) {
  if (!lean_enabled() || !lean_supported(p.h, p.f)) return false;
  if (p.f == 32) {
    if (aligned32(p.dOut)) launch<8, 1, 4>(p, s);
    else launch<4, 2, 8>(p, s);
  } else {
    launch<4, 1, 4>(p, s);
  }
  return true;
}

// The bf16 mode (gnncg_gat_fwd_bf16 / gnncg_gat_bwd_src_fused_bf16) at the same shapes: the
// lean kernels with bf16 gather tables (8 or 4 columns of one head per lane: one 16- or 8-byte
// load per lane-row), all arithmetic fp32.
#ifndef GNNCG_LEAN_FWDLP_WPC
#define GNNCG_LEAN_FWDLP_WPC 8
#endif
#ifndef GNNCG_LEAN_FWDLP_MINB
#define GNNCG_LEAN_FWDLP_MINB 4
#endif
#ifndef GNNCG_LEAN_BWDLP_WPC
#define GNNCG_LEAN_BWDLP_WPC 4
#endif
#ifndef GNNCG_LEAN_BWDLP_MINB
#define GNNCG_LEAN_BWDLP_MINB 7
#endif

bool launch_fwd_lean_lp(const GatParams& p, cudaStream_t s) {
  if (!lean_enabled() || !lean_supported(p.h, p.f) || (reinterpret_cast<uintptr_t>(p.lp) & 15)) return false;
  if (p.f == 32) {
    constexpr int W = GNNCG_LEAN_FWDLP_WPC, M = GNNCG_LEAN_FWDLP_MINB;
    const unsigned grid = lean_grid(p.num_items, W, M);
    if (p.ctr) launch_win(gat_fwd_lean_kernel<8, 8, 1, 4, W, M, true, true>, grid, W * kWarp, s, p);
    else launch_win(gat_fwd_lean_kernel<8, 8, 1, 4, W, M, false, true>, grid, W * kWarp, s, p);
  } else {
    constexpr int W = FwdShape<4>::WPC, M = FwdShape<4>::MINB;
    const unsigned grid = lean_grid(p.num_items, W, M);
    if (p.ctr) launch_win(gat_fwd_lean_kernel<8, 4, 1, 4, W, M, true, true>, grid, W * kWarp, s, p);
    else launch_win(gat_fwd_lean_kernel<8, 4, 1, 4, W, M, false, true>, grid, W * kWarp, s, p);
  }
  return true;
}

bool launch_bwd_src_lean_lp(const GatParams& p, cudaStream_t s) {
  if (!lean_enabled() || !lean_supported(p.h, p.f) || ((reinterpret_cast<uintptr_t>(p.lp) |
                                                        reinterpret_cast<uintptr_t>(p.lp_x)) & 15))
    return false;
  constexpr int W = GNNCG_LEAN_BWDLP_WPC, M = GNNCG_LEAN_BWDLP_MINB;
  const unsigned grid = lean_grid(p.num_items, W, M);
  if (p.f == 32) {
    if (p.ctr) launch_win(gat_bwd_src_lean_kernel<8, 8, 1, 4, W, M, true, true>, grid, W * kWarp, s, p);
    else launch_win(gat_bwd_src_lean_kernel<8, 8, 1, 4, W, M, false, true>, grid, W * kWarp, s, p);
  } else {
    if (p.ctr) launch_win(gat_bwd_src_lean_kernel<8, 4, 1, 4, W, M, true, true>, grid, W * kWarp, s, p);
    else launch_win(gat_bwd_src_lean_kernel<8, 4, 1, 4, W, M, false, true>, grid, W * kWarp, s, p);
  }
  return true;
}

}  // namespace gat
}  // namespace gnncg_b200
