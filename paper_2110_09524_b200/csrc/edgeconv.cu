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
// Build-time A/B knobs (scripts/build_ab.sh): edges per gather batch forward / backward, 32-byte
// column vectors, lane groups (0: one row per warp), CTAs per SM the register allocation must allow
// (4 forward / 5 backward: 64 / 48 registers, a few bytes of spill, more warps resident; C3 k = 20
// step 0.787 -> 0.749 ms, k = 40 1.077 -> 1.025 ms on one box, profiles/r02_edgeconv_ab.txt).
#ifndef GNNCG_EC_UF
#define GNNCG_EC_UF 2
#endif
#ifndef GNNCG_EC_UB
#define GNNCG_EC_UB 1
#endif
#ifndef GNNCG_EC_VW8
#define GNNCG_EC_VW8 1
#endif
#ifndef GNNCG_EC_GROUPS
#define GNNCG_EC_GROUPS 1
#endif
#ifndef GNNCG_EC_MINB_FWD
#define GNNCG_EC_MINB_FWD 4
#endif
#ifndef GNNCG_EC_MINB_BWD
#define GNNCG_EC_MINB_BWD 5
#endif

template <int VW>
struct Vec;
template <>
struct Vec<1> { using F = float; using U = uint32_t; };
template <>
struct Vec<2> { using F = float2; using U = uint2; };
template <>
struct Vec<4> { using F = float4; using U = uint4; };

// VW = 8: one 256-bit load (LDG.E.ENL2.256) of 32-byte-aligned columns.
__device__ __forceinline__ void ldv8(const void* p, uint32_t (&x)[8]) {
  asm("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7])
      : "l"(p));
}
template <int VW>
__device__ __forceinline__ void ldv(const float* p, float (&x)[VW]) {
  if constexpr (VW == 8) {
    uint32_t u[8];
    ldv8(p, u);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __uint_as_float(u[i]);
    return;
  }
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
  if constexpr (VW == 8) {
    ldv8(p, x);
    return;
  }
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

// Lane groups: L lanes own one row (VW consecutive columns each, L*VW columns per pass) and a warp
// walks 32/L rows at once, so narrow layers (C = 64 at VW = 8: 8 lanes per row, 4 rows per warp)
// keep the whole warp busy with 32-byte loads.  Every lane of a group runs its row's trip count.
// A group stages its row's neighbour and edge ids 32 at a time in its own shared-memory slot (one
// dependent id round trip per 32 edges whatever L is) and reads them back as broadcasts.
template <int L>
struct Group {
  static constexpr int SLOTS = 8 * (32 / L);  // 8 warps per CTA
  int sub, sl;
  unsigned mask;
  uint32_t* ids;  // 32 neighbour ids, then 32 edge ids
  __device__ __forceinline__ explicit Group(uint32_t* smem) {
    const int lane = threadIdx.x & 31;
    sub = lane / L;
    sl = lane % L;
    mask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (sub * L));
    ids = smem + ((threadIdx.x >> 5) * (32 / L) + sub) * 64;
  }
  __device__ __forceinline__ int64_t row() const { return ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * (32 / L) + sub; }
  __device__ __forceinline__ void stage(const uint32_t* a, const uint32_t* b, uint64_t base, int n) const {
    __syncwarp(mask);  // the previous batch is consumed
    for (int q = sl; q < n; q += L) {
      ids[q] = __ldg(a + base + q);
      ids[32 + q] = __ldg(b + base + q);
    }
    __syncwarp(mask);
  }
};

// K6: L lanes per destination row.  Rows are gathered U edges at a time: U = 2 forward, 1 backward
// (the occupancy a shallow unroll buys beats the loads in flight of U = 4: C3 k = 20 step 0.856 ->
// 0.761 ms, k = 40 1.218 -> 1.029 ms with the lane groups and 32-byte loads;
// profiles/r02_edgeconv_ab.txt).  Edges are walked in the row's (edge-id) order.
template <int VW, int L>
__global__ void __launch_bounds__(256, GNNCG_EC_MINB_FWD) edgeconv_fwd_kernel(int64_t rows, int C, int64_t row_base,
                                                           const uint64_t* __restrict__ off,
                                                           const uint32_t* __restrict__ nbr,
                                                           const uint32_t* __restrict__ eid,
                                                           const float* __restrict__ Th, int64_t ldt,
                                                           const float* __restrict__ Ph, int64_t ldp,
                                                           float* __restrict__ out, uint32_t* __restrict__ amax) {
  constexpr int U = GNNCG_EC_UF;
  __shared__ uint32_t smem[Group<L>::SLOTS * 64];
  const Group<L> grp(smem);
  const int64_t r = grp.row();
  if (r >= rows) return;
  const uint64_t e0 = off[r], e1 = off[r + 1];
  const int64_t v = row_base + r;
  for (int c0 = 0; c0 < C; c0 += L * VW) {
    const int c = c0 + grp.sl * VW;
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
      grp.stage(nbr, eid, base, n);
      for (int j = 0; j < n; j += U) {
        float x[U][VW];
#pragma unroll
        for (int t = 0; t < U; ++t) {
          const uint32_t u = grp.ids[(j + t) & 31];
          if (on && j + t < n) ldv<VW>(Th + (int64_t)u * ldt + c, x[t]);
        }
#pragma unroll
        for (int t = 0; t < U; ++t) {
          const uint32_t id = grp.ids[32 + ((j + t) & 31)];
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
// of source u, column c takes g[v, c] iff amax[v, c] == e.  L lanes per source row, VW columns per
// lane.  EAGER (the default; GNNCG_EC_EAGER=0 for the other) loads g with amax instead of after a
// match: one dependent round trip per edge instead of two, for bytes that are L2-resident here.
template <int VW, int L, bool EAGER>
__global__ void __launch_bounds__(256, GNNCG_EC_MINB_BWD) edgeconv_bwd_kernel(int64_t rows, int C, const uint64_t* __restrict__ soff,
                                                           const uint32_t* __restrict__ snbr,
                                                           const uint32_t* __restrict__ seid,
                                                           const uint64_t* __restrict__ doff,
                                                           const uint32_t* __restrict__ amax,
                                                           const float* __restrict__ g, float* __restrict__ dTh,
                                                           int64_t ldt, float* __restrict__ dPh, int64_t ldp) {
  constexpr int U = GNNCG_EC_UB;
  __shared__ uint32_t smem[Group<L>::SLOTS * 64];
  const Group<L> grp(smem);
  const int64_t u = grp.row();
  if (u >= rows) return;
  const uint64_t e0 = soff[u], e1 = soff[u + 1];
  const bool has_in = doff[u + 1] > doff[u];
  for (int c0 = 0; c0 < C; c0 += L * VW) {
    const int c = c0 + grp.sl * VW;
    const bool on = c < C;
    float acc[VW];
#pragma unroll
    for (int i = 0; i < VW; ++i) acc[i] = 0.f;
    for (uint64_t base = e0; base < e1; base += 32) {
      const int n = (int)min((uint64_t)32, e1 - base);
      grp.stage(snbr, seid, base, n);
      for (int j = 0; j < n; j += U) {
        uint32_t am[U][VW];
        float gv[U][VW];
        int64_t vv[U];
#pragma unroll
        for (int t = 0; t < U; ++t) {
          vv[t] = grp.ids[(j + t) & 31];
          if (on && j + t < n) {
            ldv<VW>(amax + vv[t] * C + c, am[t]);
            if (EAGER) ldv<VW>(g + vv[t] * C + c, gv[t]);
          }
        }
#pragma unroll
        for (int t = 0; t < U; ++t) {
          const uint32_t id = grp.ids[32 + ((j + t) & 31)];
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

// Lanes per row: the smallest of 8 / 16 / 32 covering C at VW columns per lane.
int group_lanes(int C, int vw) {
  if (!GNNCG_EC_GROUPS) return 32;
  const int need = (C + vw - 1) / vw;
  return need <= 8 ? 8 : need <= 16 ? 16 : 32;
}
unsigned group_grid(int64_t rows, int L) { return (unsigned)ceil_div(rows, (int64_t)8 * (32 / L)); }

template <int VW, int L, bool EAGER>
void launch_bwd(void* stream, const gnncg_index_t* csc, const gnncg_index_t* csr, int C, const uint32_t* amax,
                const float* g, float* dTh, int64_t ldt, float* dPh, int64_t ldp) {
  edgeconv_bwd_kernel<VW, L, EAGER><<<group_grid(csc->num_rows, L), 256, 0, as_stream(stream)>>>(
      csc->num_rows, C, csc->off, csc->nbr, csc->eid, csr->off, amax, g, dTh, ldt, dPh, ldp);
}
template <int VW, bool EAGER>
void launch_bwd_l(int L, void* stream, const gnncg_index_t* csc, const gnncg_index_t* csr, int C,
                  const uint32_t* amax, const float* g, float* dTh, int64_t ldt, float* dPh, int64_t ldp) {
  if (L == 8) launch_bwd<VW, 8, EAGER>(stream, csc, csr, C, amax, g, dTh, ldt, dPh, ldp);
  else if (L == 16) launch_bwd<VW, 16, EAGER>(stream, csc, csr, C, amax, g, dTh, ldt, dPh, ldp);
  else launch_bwd<VW, 32, EAGER>(stream, csc, csr, C, amax, g, dTh, ldt, dPh, ldp);
}
template <int VW>
void launch_fwd(int L, void* stream, const gnncg_index_t* csr, int C, int64_t row_base, const float* Th, int64_t ldt,
                const float* Ph, int64_t ldp, float* out, uint32_t* amax) {
#define GNNCG_EC_FWD(LL)                                                                                        \
  edgeconv_fwd_kernel<VW, LL><<<group_grid(csr->num_rows, LL), 256, 0, as_stream(stream)>>>(                  \
      csr->num_rows, C, row_base, csr->off, csr->nbr, csr->eid, Th, ldt, Ph, ldp, out, amax)
  if (L == 8) GNNCG_EC_FWD(8);
  else if (L == 16) GNNCG_EC_FWD(16);
  else GNNCG_EC_FWD(32);
#undef GNNCG_EC_FWD
}

bool ec_eager() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("GNNCG_EC_EAGER"); v = e ? atoi(e) : 1; }
  return v == 1;
}

// Column vector width: the widest of 8 / 4 / 2 floats per lane whose alignment holds and that still
// gives a group of 8 lanes something to do (C >= 8 VW), else the widest aligned one.
int edge_vw(int C, const void* a, int64_t lda, const void* b, int64_t ldb) {
  auto ok = [&](int w) {
    return C % w == 0 && lda % w == 0 && ldb % w == 0 && ((uintptr_t)a % (4 * w)) == 0 &&
           ((uintptr_t)b % (4 * w)) == 0;
  };
  if (!GNNCG_EC_GROUPS) {  // one row per warp
    if (GNNCG_EC_VW8 && ok(8) && C % 256 == 0) return 8;
    return ok(4) && C >= 128 ? 4 : ok(2) && C >= 64 ? 2 : 1;
  }
  for (int w = GNNCG_EC_VW8 ? 8 : 4; w > 1; w /= 2)
    if (ok(w) && C >= 8 * w) return w;
  for (int w = GNNCG_EC_VW8 ? 8 : 4; w > 1; w /= 2)
    if (ok(w)) return w;
  return 1;
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
  const int vw = edge_vw(C, Th, ldt, Ph, ldp);
  const int L = group_lanes(C, vw);
  if (vw == 8) launch_fwd<8>(L, stream, csr, C, row_base, Th, ldt, Ph, ldp, out, amax);
  else if (vw == 4) launch_fwd<4>(L, stream, csr, C, row_base, Th, ldt, Ph, ldp, out, amax);
  else if (vw == 2) launch_fwd<2>(L, stream, csr, C, row_base, Th, ldt, Ph, ldp, out, amax);
  else launch_fwd<1>(L, stream, csr, C, row_base, Th, ldt, Ph, ldp, out, amax);
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
  // (amax and g are dense C-wide rows: their alignment follows from C and the base pointers)
  int vw = edge_vw(C, dTh, ldt, dPh, ldp);
  while (vw > 1 && (((uintptr_t)amax % (4 * vw)) || ((uintptr_t)g % (4 * vw)))) vw /= 2;
  const int L = group_lanes(C, vw);
#define GNNCG_EC_BWD(W)                                                                                    \
  (ec_eager() ? launch_bwd_l<W, true>(L, stream, csc, csr, C, amax, g, dTh, ldt, dPh, ldp)                    \
              : launch_bwd_l<W, false>(L, stream, csc, csr, C, amax, g, dTh, ldt, dPh, ldp))
  if (vw == 8) GNNCG_EC_BWD(8);
  else if (vw == 4) GNNCG_EC_BWD(4);
  else if (vw == 2) GNNCG_EC_BWD(2);
  else GNNCG_EC_BWD(1);
#undef GNNCG_EC_BWD
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

}  // extern "C"
