// SPDX-License-Identifier: Apache-2.0
//
// oracle/oracle.cpp -- TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference's fused-GNN-layer semantics, used (a) as the
// parity checker by tests/, __graft_entry__.smoke() and (b) as the timed CPU
// baseline leg of bench.py.  Nothing in the product package links or calls this
// library; the product path fails loudly when its CUDA extension is missing.
//
// The reference ships no code for the GAT / EdgeConv / GMMConv layers (ir.cpp,
// passes.cpp, executor.cpp and reference.cpp are absent: proj/CMakeLists.txt:19-23),
// so the layer math is restated from the specification and the paper:
//   * graph index        : proj/src/graph.cpp:14-28 (counting sort, rows by edge id)
//   * dense transforms   : proj/src/tensor.cpp:8-60 (matmul / matmul_nt / matmul_tn)
//   * LeakyReLU(0.2)     : proj/include/gnncg/tensor.hpp:75,93 
//   * head-major layout  : proj/include/gnncg/tensor.hpp:17-19,99-121 
//   * GAT layer          : PAPER.md:543-558 (App. A.2), edge-softmax RS1/RS2 PAPER.md:527-530
//   * EdgeConv layer     : PAPER.md:562-582 ; tie-break / empty rows SPEC.md:212-213
//   * GMMConv layer      : PAPER.md:591-605 ; diagonal Sigma SPEC.md:216
//   * backward rules     : PAPER.md:615-662 (App. B) ; loss = sum of exits SPEC.md:217
//   * executor semantics : SPEC.md:335-360 (vertex_balanced, recompute backward)
//
// Two flavours are provided:
//   *_f64  : serial, "stash everything" per-edge chain rule in double precision.
//            This is the parity oracle (f64 is the oracle precision).
//   *_f32_omp : the SPEC executor restated for speed -- vertex_balanced OpenMP over
//            destination rows, recompute-based two-pass backward
//            (SPEC.md:276,355), f32.  This is the timed CPU baseline ("port").
//
// Index layout (identical to gnncg::AdjIndex split to SoA, graph.hpp:19-29):
//   off[V+1] (u64), nbr[E] (u32 = AdjEntry::vertex), eid[E] (u32 = AdjEntry::edge).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef std::uint64_t u64;
typedef std::uint32_t u32;
typedef std::int64_t i64;

namespace {

template <typename T>
inline T lrelu(T z, T slope) { return z > T(0) ? z : slope * z; }  // tensor.hpp:75
template <typename T>
inline T lrelu_grad(T z, T slope) { return z > T(0) ? T(1) : slope; }

// C[M,N] = A[M,K] * B[K,N]   (tensor.cpp:8-24 loop order: i, k, j)
template <typename T>
void mm_nn(u64 M, u64 K, u64 N, const T* A, const T* B, T* C) {
#pragma omp parallel for schedule(static)
  for (i64 i = 0; i < (i64)M; ++i) {
    T* c = C + (u64)i * N;
    for (u64 j = 0; j < N; ++j) c[j] = T(0);
    const T* a = A + (u64)i * K;
    for (u64 k = 0; k < K; ++k) {
      const T aik = a[k];
      const T* b = B + k * N;
      for (u64 j = 0; j < N; ++j) c[j] += aik * b[j];
    }
  }
}

// C[M,N] = A[M,K] * B[N,K]^T   (tensor.cpp:26-42)
template <typename T>
void mm_nt(u64 M, u64 K, u64 N, const T* A, const T* B, T* C) {
#pragma omp parallel for schedule(static)
  for (i64 i = 0; i < (i64)M; ++i) {
    const T* a = A + (u64)i * K;
    for (u64 j = 0; j < N; ++j) {
      const T* b = B + j * K;
      T acc = T(0);
      for (u64 k = 0; k < K; ++k) acc += a[k] * b[k];
      C[(u64)i * N + j] = acc;
    }
  }
}

// C[M,N] = A[K,M]^T * B[K,N]   (tensor.cpp:44-60)
template <typename T>
void mm_tn(u64 K, u64 M, u64 N, const T* A, const T* B, T* C) {
#pragma omp parallel for schedule(static)
  for (i64 i = 0; i < (i64)M; ++i) {
    T* c = C + (u64)i * N;
    for (u64 j = 0; j < N; ++j) c[j] = T(0);
    for (u64 k = 0; k < K; ++k) {
      const T aki = A[k * M + (u64)i];
      const T* b = B + k * N;
      for (u64 j = 0; j < N; ++j) c[j] += aki * b[j];
    }
  }
}

// A_l[v,k] = <Ht[v,k,:], a_l[k,:]>  (reorganized LPs, SPEC.md:258,262 )
template <typename T>
void attn_dots(u64 V, int h, int f, const T* Ht, const T* a, T* A) {
  const u64 hf = (u64)h * f;
#pragma omp parallel for schedule(static)
  for (i64 v = 0; v < (i64)V; ++v) {
    for (int k = 0; k < h; ++k) {
      T s = T(0);
      for (int j = 0; j < f; ++j) s += Ht[(u64)v * hf + (u64)k * f + j] * a[(u64)k * f + j];
      A[(u64)v * h + k] = s;
    }
  }
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------------------
// Graph index: restatement of build_index (graph.cpp:14-28).  Rows keyed by
// key[e]; entries filled in ascending edge id, so every row is sorted by edge id.
// ---------------------------------------------------------------------------
void orc_build_index(u64 V, u64 E, const u32* key, const u32* other, u64* off, u32* nbr, u32* eid) {
  for (u64 v = 0; v <= V; ++v) off[v] = 0;
  for (u64 e = 0; e < E; ++e) off[(u64)key[e] + 1]++;
  for (u64 v = 0; v < V; ++v) off[v + 1] += off[v];
  std::vector<u64> cur(off, off + V);
  for (u64 e = 0; e < E; ++e) {
    const u64 p = cur[key[e]]++;
    nbr[p] = other[e];
    eid[p] = (u32)e;
  }
}

// Row-block partitioner (new; north_star + SURVEY §8a a5): P contiguous
// destination-row blocks balanced by edge count.  bound[p] = lower_bound(off, ceil(p*E/P)).
void orc_partition_rows(u64 V, const u64* off, int P, u64* bound) {
  const u64 E = off[V];
  bound[0] = 0;
  for (int p = 1; p < P; ++p) {
    const u64 target = ((u64)p * E + (u64)P - 1) / (u64)P;
    bound[p] = (u64)(std::lower_bound(off, off + V + 1, target) - off);
    if (bound[p] > V) bound[p] = V;
    if (bound[p] < bound[p - 1]) bound[p] = bound[p - 1];
  }
  bound[P] = V;
}

// Dense helpers exposed for tests (f64).
void orc_mm_nn_f64(u64 M, u64 K, u64 N, const double* A, const double* B, double* C) { mm_nn(M, K, N, A, B, C); }
void orc_mm_nt_f64(u64 M, u64 K, u64 N, const double* A, const double* B, double* C) { mm_nt(M, K, N, A, B, C); }
void orc_mm_tn_f64(u64 K, u64 M, u64 N, const double* A, const double* B, double* C) { mm_tn(K, M, N, A, B, C); }
void orc_mm_nn_f32(u64 M, u64 K, u64 N, const float* A, const float* B, float* C) { mm_nn(M, K, N, A, B, C); }
void orc_mm_nt_f32(u64 M, u64 K, u64 N, const float* A, const float* B, float* C) { mm_nt(M, K, N, A, B, C); }
void orc_mm_tn_f32(u64 K, u64 M, u64 N, const float* A, const float* B, float* C) { mm_tn(K, M, N, A, B, C); }

// Dense-adjacency oracle for Aggregate(sum, x w_e, copy_u):
// out[v] = sum_u A[u][v] * H[u]   with A the multiplicity matrix and unit weights.
void orc_dense_aggregate_f64(u64 V, u64 E, const u32* src, const u32* dst, const double* w, int F,
                             const double* H, double* out) {
  std::vector<double> A(V * V, 0.0);
  for (u64 e = 0; e < E; ++e) A[(u64)src[e] * V + dst[e]] += (w ? w[e] : 1.0);
  for (u64 v = 0; v < V; ++v)
    for (int j = 0; j < F; ++j) {
      double s = 0.0;
      for (u64 u = 0; u < V; ++u) s += A[u * V + v] * H[u * (u64)F + j];
      out[v * (u64)F + j] = s;
    }
}

// ---------------------------------------------------------------------------
// GAT fused region, forward (PAPER.md:543-558 ).
//   s_e = LReLU(A_l[u] + A_r[v]) ; m = max_e s_e ; d = sum_e exp(s_e - m)
//   out[v,k,:] = sum_e exp(s_e - m)/d * Ht[u,k,:]
// Empty in-neighbourhood: out = 0, m = d = 0.
// ---------------------------------------------------------------------------
void orc_gat_region_fwd_f64(u64 V, const u64* off, const u32* src, const double* Ht, const double* Al,
                            const double* Ar, int h, int f, double slope, double* out, double* m, double* d) {
  const u64 hf = (u64)h * f;
  for (u64 v = 0; v < V; ++v) {
    double* o = out + v * hf;
    for (u64 j = 0; j < hf; ++j) o[j] = 0.0;
    for (int k = 0; k < h; ++k) {
      if (off[v] == off[v + 1]) {
        m[v * h + k] = 0.0;
        d[v * h + k] = 0.0;
        continue;
      }
      double mx = -std::numeric_limits<double>::infinity();
      for (u64 i = off[v]; i < off[v + 1]; ++i) mx = std::max(mx, lrelu(Al[(u64)src[i] * h + k] + Ar[v * h + k], slope));
      double den = 0.0;
      for (u64 i = off[v]; i < off[v + 1]; ++i) den += std::exp(lrelu(Al[(u64)src[i] * h + k] + Ar[v * h + k], slope) - mx);
      for (u64 i = off[v]; i < off[v + 1]; ++i) {
        const u64 u = src[i];
        const double a = std::exp(lrelu(Al[u * h + k] + Ar[v * h + k], slope) - mx) / den;
        for (int j = 0; j < f; ++j) o[(u64)k * f + j] += a * Ht[u * hf + (u64)k * f + j];
      }
      m[v * h + k] = mx;
      d[v * h + k] = den;
    }
  }
}

// Full GAT layer forward in f64: Ht = H W ; A_l, A_r ; fused region.
void orc_gat_layer_fwd_f64(u64 V, const u64* off, const u32* src, u64 Fin, const double* H, const double* W,
                           const double* al, const double* ar, int h, int f, double slope, double* Ht,
                           double* Al, double* Ar, double* out, double* m, double* d) {
  const u64 hf = (u64)h * f;
  mm_nn(V, Fin, hf, H, W, Ht);
  attn_dots(V, h, f, Ht, al, Al);
  attn_dots(V, h, f, Ht, ar, Ar);
  orc_gat_region_fwd_f64(V, off, src, Ht, Al, Ar, h, f, slope, out, m, d);
}

// GAT region backward, f64, "stash everything" per-edge chain rule (App. B,
// PAPER.md:615-662).  Iterates destination rows in CSR order; per-edge alpha is
// materialised (row-local) rather than recomputed -- an independent derivation
// from the GPU's two-pass recompute dataflow.
//   outputs: dHt (V x hf, includes the A_l/A_r LP back-prop), dAl, dAr (V x h),
//            dal, dar (h x f)
void orc_gat_region_bwd_f64(u64 V, const u64* off, const u32* src, const double* Ht, const double* Al,
                            const double* Ar, const double* al, const double* ar, int h, int f, double slope,
                            const double* dOut, double* dHt, double* dAl, double* dAr, double* dal, double* dar) {
  const u64 hf = (u64)h * f;
  std::fill(dHt, dHt + V * hf, 0.0);
  std::fill(dAl, dAl + V * h, 0.0);
  std::fill(dAr, dAr + V * h, 0.0);
  std::vector<double> alpha, dalpha, z;
  for (u64 v = 0; v < V; ++v) {
    const u64 b = off[v], e = off[v + 1], n = e - b;
    if (n == 0) continue;
    for (int k = 0; k < h; ++k) {
      alpha.assign(n, 0.0);
      dalpha.assign(n, 0.0);
      z.assign(n, 0.0);
      double mx = -std::numeric_limits<double>::infinity();
      for (u64 i = 0; i < n; ++i) {
        z[i] = Al[(u64)src[b + i] * h + k] + Ar[v * h + k];
        mx = std::max(mx, lrelu(z[i], slope));
      }
      double den = 0.0;
      for (u64 i = 0; i < n; ++i) den += std::exp(lrelu(z[i], slope) - mx);
      double c = 0.0;
      for (u64 i = 0; i < n; ++i) {
        const u64 u = src[b + i];
        alpha[i] = std::exp(lrelu(z[i], slope) - mx) / den;
        double da = 0.0;  // d alpha_e = <dOut[v,k,:], Ht[u,k,:]>
        for (int j = 0; j < f; ++j) da += dOut[v * hf + (u64)k * f + j] * Ht[u * hf + (u64)k * f + j];
        dalpha[i] = da;
        c += alpha[i] * da;
        // Aggregate backward: dHt[u] += alpha * dOut[v]   (Scatter(copy_v) + ApplyEdge)
        for (int j = 0; j < f; ++j) dHt[u * hf + (u64)k * f + j] += alpha[i] * dOut[v * hf + (u64)k * f + j];
      }
      for (u64 i = 0; i < n; ++i) {
        const u64 u = src[b + i];
        const double ds = alpha[i] * (dalpha[i] - c);  // softmax backward
        const double dz = ds * lrelu_grad(z[i], slope);
        dAl[u * h + k] += dz;  // Scatter(u_add_v) backward: Gather over adjacent edges
        dAr[v * h + k] += dz;
      }
    }
  }
  // LP backward: A_l = Ht . a_l  =>  dHt += dAl (x) a_l ; da_l = sum_v dAl[v,k] Ht[v,k,:]
  std::fill(dal, dal + hf, 0.0);
  std::fill(dar, dar + hf, 0.0);
  for (u64 v = 0; v < V; ++v)
    for (int k = 0; k < h; ++k)
      for (int j = 0; j < f; ++j) {
        const u64 c = v * hf + (u64)k * f + j;
        dal[(u64)k * f + j] += dAl[v * h + k] * Ht[c];
        dar[(u64)k * f + j] += dAr[v * h + k] * Ht[c];
      }
  for (u64 v = 0; v < V; ++v)
    for (int k = 0; k < h; ++k)
      for (int j = 0; j < f; ++j)
        dHt[v * hf + (u64)k * f + j] += dAl[v * h + k] * al[(u64)k * f + j] + dAr[v * h + k] * ar[(u64)k * f + j];
}

// Full GAT layer backward in f64.  dH may be null (first layer).
void orc_gat_layer_bwd_f64(u64 V, const u64* off, const u32* src, u64 Fin, const double* H, const double* W,
                           const double* al, const double* ar, int h, int f, double slope, const double* Ht,
                           const double* Al, const double* Ar, const double* dOut, double* dH, double* dW,
                           double* dal, double* dar, double* dHt, double* dAl, double* dAr) {
  const u64 hf = (u64)h * f;
  orc_gat_region_bwd_f64(V, off, src, Ht, Al, Ar, al, ar, h, f, slope, dOut, dHt, dAl, dAr, dal, dar);
  mm_tn(V, Fin, hf, H, dHt, dW);          // dW = H^T dHt      (tensor.cpp:44-60)
  if (dH) mm_nt(V, hf, Fin, dHt, W, dH);  // dH = dHt W^T      (tensor.cpp:26-42)
}

// ---------------------------------------------------------------------------
// GAT, the SPEC executor restated for speed: vertex_balanced OpenMP over
// destination rows, stash m, d only, recompute the
// O(|E|) edge values in backward.  T = float: the timed CPU baseline
// (*_f32_omp); T = double: the parity oracle at benchmark scale (*_f64_omp) -- the
// serial stash-everything *_f64 above is the independent derivation it is checked
// against on small graphs (tests/test_oracle.py).
// ---------------------------------------------------------------------------
}  // extern "C"
namespace {
template <typename T>
void gat_region_fwd_omp(u64 V, const u64* off, const u32* src, const T* Ht, const T* Al, const T* Ar, int h, int f,
                        T slope, T* out, T* m, T* d) {
  const u64 hf = (u64)h * f;
#pragma omp parallel for schedule(dynamic, 64)
  for (i64 vv = 0; vv < (i64)V; ++vv) {
    const u64 v = (u64)vv;
    T* o = out + v * hf;
    for (u64 j = 0; j < hf; ++j) o[j] = T(0);
    for (int k = 0; k < h; ++k) {
      const T ar_ = Ar[v * h + k];
      T mx = -std::numeric_limits<T>::infinity(), den = T(0);
      for (u64 i = off[v]; i < off[v + 1]; ++i) mx = std::max(mx, lrelu(Al[(u64)src[i] * h + k] + ar_, slope));
      for (u64 i = off[v]; i < off[v + 1]; ++i) {
        const u64 u = src[i];
        const T p = std::exp(lrelu(Al[u * h + k] + ar_, slope) - mx);
        den += p;
        const T* x = Ht + u * hf + (u64)k * f;
        for (int j = 0; j < f; ++j) o[(u64)k * f + j] += p * x[j];
      }
      if (off[v] == off[v + 1]) { mx = T(0); den = T(0); }
      const T inv = den > T(0) ? T(1) / den : T(0);
      for (int j = 0; j < f; ++j) o[(u64)k * f + j] *= inv;
      m[v * h + k] = mx;
      d[v * h + k] = den;
    }
  }
}

// Backward, two passes without atomics:
//  pass 1 (csr_dst, per v):  c[v] = sum alpha*dalpha ; dAr[v] = sum dz
//  pass 2 (csc_src, per u):  dAl[u] = sum dz ; dHt[u] = sum alpha * dOut[v]  (+ LP terms)
template <typename T>
void gat_region_bwd_omp(u64 V, const u64* doff, const u32* dsrc, const u64* soff, const u32* sdst, const T* Ht,
                        const T* Al, const T* Ar, const T* al, const T* ar, int h, int f, T slope, const T* m,
                        const T* d, const T* dOut, T* dHt, T* dAl, T* dAr, T* c, T* dal, T* dar) {
  const u64 hf = (u64)h * f;
#pragma omp parallel for schedule(dynamic, 64)
  for (i64 vv = 0; vv < (i64)V; ++vv) {
    const u64 v = (u64)vv;
    for (int k = 0; k < h; ++k) {
      T cc = T(0), P = T(0), Q = T(0);
      const T inv = d[v * h + k] > T(0) ? T(1) / d[v * h + k] : T(0);
      const T* g = dOut + v * hf + (u64)k * f;
      for (u64 i = doff[v]; i < doff[v + 1]; ++i) {
        const u64 u = dsrc[i];
        const T z = Al[u * h + k] + Ar[v * h + k];
        const T a = std::exp(lrelu(z, slope) - m[v * h + k]) * inv;
        const T* x = Ht + u * hf + (u64)k * f;
        T da = T(0);
        for (int j = 0; j < f; ++j) da += g[j] * x[j];
        const T ga = lrelu_grad(z, slope) * a;
        cc += a * da;
        P += ga * da;
        Q += ga;
      }
      c[v * h + k] = cc;
      dAr[v * h + k] = P - cc * Q;
    }
  }
#pragma omp parallel for schedule(dynamic, 64)
  for (i64 uu = 0; uu < (i64)V; ++uu) {
    const u64 u = (u64)uu;
    T* o = dHt + u * hf;
    for (u64 j = 0; j < hf; ++j) o[j] = T(0);
    for (int k = 0; k < h; ++k) {
      T sdz = T(0);
      const T* x = Ht + u * hf + (u64)k * f;
      for (u64 i = soff[u]; i < soff[u + 1]; ++i) {
        const u64 v = sdst[i];
        const T z = Al[u * h + k] + Ar[v * h + k];
        const T inv = d[v * h + k] > T(0) ? T(1) / d[v * h + k] : T(0);
        const T a = std::exp(lrelu(z, slope) - m[v * h + k]) * inv;
        const T* g = dOut + v * hf + (u64)k * f;
        T da = T(0);
        for (int j = 0; j < f; ++j) da += g[j] * x[j];
        sdz += lrelu_grad(z, slope) * a * (da - c[v * h + k]);
        for (int j = 0; j < f; ++j) o[(u64)k * f + j] += a * g[j];
      }
      dAl[u * h + k] = sdz;
    }
    for (int k = 0; k < h; ++k)
      for (int j = 0; j < f; ++j)
        o[(u64)k * f + j] += dAl[u * h + k] * al[(u64)k * f + j] + dAr[u * h + k] * ar[(u64)k * f + j];
  }
  // da_l[k,j] = sum_v dAl[v,k] Ht[v,k,j]: columns in parallel, rows in order (deterministic)
#pragma omp parallel for schedule(static)
  for (i64 jj = 0; jj < (i64)hf; ++jj) {
    const u64 j = (u64)jj, k = j / (u64)f;
    T sl = T(0), sr = T(0);
    for (u64 v = 0; v < V; ++v) {
      sl += dAl[v * h + k] * Ht[v * hf + j];
      sr += dAr[v * h + k] * Ht[v * hf + j];
    }
    dal[j] = sl;
    dar[j] = sr;
  }
}

template <typename T>
void gat_layer_fwd_omp(u64 V, const u64* off, const u32* src, u64 Fin, const T* H, const T* W, const T* al,
                       const T* ar, int h, int f, T slope, T* Ht, T* Al, T* Ar, T* out, T* m, T* d) {
  const u64 hf = (u64)h * f;
  mm_nn(V, Fin, hf, H, W, Ht);
  attn_dots(V, h, f, Ht, al, Al);
  attn_dots(V, h, f, Ht, ar, Ar);
  gat_region_fwd_omp(V, off, src, Ht, Al, Ar, h, f, slope, out, m, d);
}

template <typename T>
void gat_layer_bwd_omp(u64 V, const u64* doff, const u32* dsrc, const u64* soff, const u32* sdst, u64 Fin,
                       const T* H, const T* W, const T* al, const T* ar, int h, int f, T slope, const T* Ht,
                       const T* Al, const T* Ar, const T* m, const T* d, const T* dOut, T* dH, T* dW, T* dal, T* dar,
                       T* dHt, T* dAl, T* dAr, T* c) {
  const u64 hf = (u64)h * f;
  gat_region_bwd_omp(V, doff, dsrc, soff, sdst, Ht, Al, Ar, al, ar, h, f, slope, m, d, dOut, dHt, dAl, dAr, c, dal,
                     dar);
  mm_tn(V, Fin, hf, H, dHt, dW);
  if (dH) mm_nt(V, hf, Fin, dHt, W, dH);
}
}  // namespace
extern "C" {

#define ORC_GAT_OMP(SUF, T)                                                                                          \
  void orc_gat_region_fwd_##SUF(u64 V, const u64* off, const u32* src, const T* Ht, const T* Al, const T* Ar, int h, \
                                int f, T slope, T* out, T* m, T* d) {                                               \
    gat_region_fwd_omp<T>(V, off, src, Ht, Al, Ar, h, f, slope, out, m, d);                                         \
  }                                                                                                                  \
  void orc_gat_region_bwd_##SUF(u64 V, const u64* doff, const u32* dsrc, const u64* soff, const u32* sdst,          \
                                const T* Ht, const T* Al, const T* Ar, const T* al, const T* ar, int h, int f,       \
                                T slope, const T* m, const T* d, const T* dOut, T* dHt, T* dAl, T* dAr, T* c,        \
                                T* dal, T* dar) {                                                                    \
    gat_region_bwd_omp<T>(V, doff, dsrc, soff, sdst, Ht, Al, Ar, al, ar, h, f, slope, m, d, dOut, dHt, dAl, dAr, c,  \
                          dal, dar);                                                                                 \
  }                                                                                                                  \
  void orc_gat_layer_fwd_##SUF(u64 V, const u64* off, const u32* src, u64 Fin, const T* H, const T* W, const T* al,  \
                               const T* ar, int h, int f, T slope, T* Ht, T* Al, T* Ar, T* out, T* m, T* d) {        \
    gat_layer_fwd_omp<T>(V, off, src, Fin, H, W, al, ar, h, f, slope, Ht, Al, Ar, out, m, d);                       \
  }                                                                                                                  \
  void orc_gat_layer_bwd_##SUF(u64 V, const u64* doff, const u32* dsrc, const u64* soff, const u32* sdst, u64 Fin,  \
                               const T* H, const T* W, const T* al, const T* ar, int h, int f, T slope, const T* Ht, \
                               const T* Al, const T* Ar, const T* m, const T* d, const T* dOut, T* dH, T* dW,       \
                               T* dal, T* dar, T* dHt, T* dAl, T* dAr, T* c) {                                       \
    gat_layer_bwd_omp<T>(V, doff, dsrc, soff, sdst, Fin, H, W, al, ar, h, f, slope, Ht, Al, Ar, m, d, dOut, dH, dW,  \
                         dal, dar, dHt, dAl, dAr, c);                                                                \
  }

ORC_GAT_OMP(f32_omp, float)
ORC_GAT_OMP(f64_omp, double)
#undef ORC_GAT_OMP

// ---------------------------------------------------------------------------
// EdgeConv (reorganized per SPEC.md:261):
//   out[v,c] = max_{(u,e) in in(v)} ((Th[u,c] - Th[v,c]) + Ph[v,c])
//   argmax[v,c] = edge id of the first (lowest-eid) edge attaining the max
//   empty row: out = 0, argmax = 0xFFFFFFFF (the "degree-0 mask")
// f32 version evaluates exactly the stated expression in round-to-nearest with
// a strict '>' in row (= edge id) order -- the bit-exact argmax contract.
// ---------------------------------------------------------------------------
}  // extern "C"
template <typename T>
static void edgeconv_fwd(u64 V, const u64* off, const u32* src, const u32* eid, int C, const T* Th, const T* Ph,
                         T* out, u32* amax) {
#pragma omp parallel for schedule(dynamic, 64)
  for (i64 vv = 0; vv < (i64)V; ++vv) {
    const u64 v = (u64)vv;
    for (int c = 0; c < C; ++c) {
      const u64 vc = v * C + c;
      if (off[v] == off[v + 1]) {
        out[vc] = T(0);
        amax[vc] = 0xFFFFFFFFu;
        continue;
      }
      T best = T(0);
      u32 arg = 0xFFFFFFFFu;
      for (u64 i = off[v]; i < off[v + 1]; ++i) {
        volatile T diff = Th[(u64)src[i] * C + c] - Th[vc];  // volatile: forbid reassociation/contraction
        volatile T val = diff + Ph[vc];
        if (arg == 0xFFFFFFFFu || val > best) {
          best = val;
          arg = eid[i];
        }
      }
      out[vc] = best;
      amax[vc] = arg;
    }
  }
}

extern "C" {
void orc_edgeconv_fwd_f32(u64 V, const u64* off, const u32* src, const u32* eid, int C, const float* Th,
                          const float* Ph, float* out, u32* amax) {
  edgeconv_fwd(V, off, src, eid, C, Th, Ph, out, amax);
}
void orc_edgeconv_fwd_f64(u64 V, const u64* off, const u32* src, const u32* eid, int C, const double* Th,
                          const double* Ph, double* out, u32* amax) {
  edgeconv_fwd(V, off, src, eid, C, Th, Ph, out, amax);
}

// Gather(max) backward = argmax routing:
//   dTh[src(argmax)] += g ; dTh[v] -= g ; dPh[v] += g   (rows with deg > 0 only)
// edge_src[e] maps an edge id to its source (Graph::edge_src, graph.hpp:48).
}  // extern "C"
template <typename T>
static void edgeconv_bwd(u64 V, const u64* off, const u32* edge_src, int C, const u32* amax, const T* g, T* dTh,
                         T* dPh) {
  std::fill(dTh, dTh + V * C, T(0));
  std::fill(dPh, dPh + V * C, T(0));
  for (u64 v = 0; v < V; ++v) {
    if (off[v] == off[v + 1]) continue;
    for (int c = 0; c < C; ++c) {
      const u64 vc = v * C + c;
      dTh[(u64)edge_src[amax[vc]] * C + c] += g[vc];
      dTh[vc] -= g[vc];
      dPh[vc] += g[vc];
    }
  }
}
extern "C" {
void orc_edgeconv_bwd_f64(u64 V, const u64* off, const u32* edge_src, int C, const u32* amax, const double* g,
                          double* dTh, double* dPh) {
  edgeconv_bwd(V, off, edge_src, C, amax, g, dTh, dPh);
}
void orc_edgeconv_bwd_f32(u64 V, const u64* off, const u32* edge_src, int C, const u32* amax, const float* g,
                          float* dTh, float* dPh) {
  edgeconv_bwd(V, off, edge_src, C, amax, g, dTh, dPh);
}

// Layer-level EdgeConv f64: Th = H Theta, Ph = H Phi (Theta, Phi given Fin x C).
void orc_edgeconv_layer_fwd_f64(u64 V, const u64* off, const u32* src, const u32* eid, u64 Fin, const double* H,
                                const double* Theta, const double* Phi, int C, double* Th, double* Ph, double* out,
                                u32* amax) {
  mm_nn(V, Fin, (u64)C, H, Theta, Th);
  mm_nn(V, Fin, (u64)C, H, Phi, Ph);
  edgeconv_fwd(V, off, src, eid, C, Th, Ph, out, amax);
}
void orc_edgeconv_layer_bwd_f64(u64 V, const u64* off, const u32* edge_src, u64 Fin, const double* H,
                                const double* Theta, const double* Phi, int C, const u32* amax, const double* g,
                                double* dH, double* dTheta, double* dPhi, double* dTh, double* dPh) {
  edgeconv_bwd(V, off, edge_src, C, amax, g, dTh, dPh);
  mm_tn(V, Fin, (u64)C, H, dTh, dTheta);
  mm_tn(V, Fin, (u64)C, H, dPh, dPhi);
  if (dH) {
    std::vector<double> t((size_t)(V * Fin));
    mm_nt(V, (u64)C, Fin, dTh, Theta, dH);
    mm_nt(V, (u64)C, Fin, dPh, Phi, t.data());
    for (u64 i = 0; i < V * Fin; ++i) dH[i] += t[i];
  }
}

// ---------------------------------------------------------------------------
// GMMConv (PAPER.md:591-605 ; SPEC.md:216 diagonal Sigma).  Parameterisation
// recorded in DESIGN.md: Sigma_k^{-1} = diag(sinv_k^2) with sinv the learned
// inverse standard deviation; pseudo-coordinates m_uv = H[u] P_l + H[v] P_r
// (linear f reorganized to two ApplyVertex + u_add_v).
//   hW = H W (V x K*f) ; pl = H P_l ; pr = H P_r (V x r)
//   w_k(m) = exp(-1/2 sum_d (m_d - mu_kd)^2 sinv_kd^2)
//   out[v] = (1/K) sum_u sum_k w_k(pl[u] + pr[v]) hW[u,k,:]
// ---------------------------------------------------------------------------
void orc_gmm_region_fwd_f64(u64 V, const u64* off, const u32* src, int K, int r, int f, const double* hW,
                            const double* pl, const double* pr, const double* mu, const double* sinv, double* out) {
  const u64 Kf = (u64)K * f;
  std::vector<double> w(K);
  for (u64 v = 0; v < V; ++v) {
    double* o = out + v * f;
    for (int j = 0; j < f; ++j) o[j] = 0.0;
    for (u64 i = off[v]; i < off[v + 1]; ++i) {
      const u64 u = src[i];
      for (int k = 0; k < K; ++k) {
        double q = 0.0;
        for (int t = 0; t < r; ++t) {
          const double md = pl[u * r + t] + pr[v * r + t] - mu[k * r + t];
          const double s = sinv[k * r + t];
          q += md * md * s * s;
        }
        w[k] = std::exp(-0.5 * q);
      }
      for (int k = 0; k < K; ++k)
        for (int j = 0; j < f; ++j) o[j] += w[k] * hW[u * Kf + (u64)k * f + j] / (double)K;
    }
  }
}

// Backward (stash-everything chain rule).  Outputs d hW, d pl, d pr, dmu, dsinv.
void orc_gmm_region_bwd_f64(u64 V, const u64* off, const u32* src, int K, int r, int f, const double* hW,
                            const double* pl, const double* pr, const double* mu, const double* sinv,
                            const double* dOut, double* dhW, double* dpl, double* dpr, double* dmu, double* dsinv) {
  const u64 Kf = (u64)K * f;
  std::fill(dhW, dhW + V * Kf, 0.0);
  std::fill(dpl, dpl + V * r, 0.0);
  std::fill(dpr, dpr + V * r, 0.0);
  std::fill(dmu, dmu + (u64)K * r, 0.0);
  std::fill(dsinv, dsinv + (u64)K * r, 0.0);
  std::vector<double> w(K), md((size_t)K * r);
  for (u64 v = 0; v < V; ++v) {
    const double* g = dOut + v * f;
    for (u64 i = off[v]; i < off[v + 1]; ++i) {
      const u64 u = src[i];
      for (int k = 0; k < K; ++k) {
        double q = 0.0;
        for (int t = 0; t < r; ++t) {
          md[k * r + t] = pl[u * r + t] + pr[v * r + t] - mu[k * r + t];
          const double s = sinv[k * r + t];
          q += md[k * r + t] * md[k * r + t] * s * s;
        }
        w[k] = std::exp(-0.5 * q);
      }
      for (int k = 0; k < K; ++k) {
        double dw = 0.0;
        for (int j = 0; j < f; ++j) {
          dw += g[j] * hW[u * Kf + (u64)k * f + j] / (double)K;
          dhW[u * Kf + (u64)k * f + j] += w[k] * g[j] / (double)K;
        }
        // w = exp(-q/2): dq = -w/2 * dw ; q = sum md^2 s^2
        const double dq = -0.5 * w[k] * dw;
        for (int t = 0; t < r; ++t) {
          const double s = sinv[k * r + t], x = md[k * r + t];
          const double dmd = dq * 2.0 * x * s * s;
          dsinv[k * r + t] += dq * 2.0 * x * x * s;
          dmu[k * r + t] -= dmd;
          dpl[u * r + t] += dmd;
          dpr[v * r + t] += dmd;
        }
      }
    }
  }
}

// Layer-level GMM f64.  Params: W (Fin x K*f), Pl, Pr (Fin x r), mu, sinv (K x r).
void orc_gmm_layer_fwd_f64(u64 V, const u64* off, const u32* src, u64 Fin, const double* H, const double* W,
                           const double* Pl, const double* Pr, const double* mu, const double* sinv, int K, int r,
                           int f, double* hW, double* pl, double* pr, double* out) {
  mm_nn(V, Fin, (u64)K * f, H, W, hW);
  mm_nn(V, Fin, (u64)r, H, Pl, pl);
  mm_nn(V, Fin, (u64)r, H, Pr, pr);
  orc_gmm_region_fwd_f64(V, off, src, K, r, f, hW, pl, pr, mu, sinv, out);
}

void orc_gmm_layer_bwd_f64(u64 V, const u64* off, const u32* src, u64 Fin, const double* H, const double* W,
                           const double* Pl, const double* Pr, const double* mu, const double* sinv, int K, int r,
                           int f, const double* hW, const double* pl, const double* pr, const double* dOut,
                           double* dH, double* dW, double* dPl, double* dPr, double* dmu, double* dsinv,
                           double* dhW, double* dpl, double* dpr) {
  const u64 Kf = (u64)K * f;
  orc_gmm_region_bwd_f64(V, off, src, K, r, f, hW, pl, pr, mu, sinv, dOut, dhW, dpl, dpr, dmu, dsinv);
  mm_tn(V, Fin, Kf, H, dhW, dW);
  mm_tn(V, Fin, (u64)r, H, dpl, dPl);
  mm_tn(V, Fin, (u64)r, H, dpr, dPr);
  if (dH) {
    std::vector<double> t((size_t)(V * Fin));
    mm_nt(V, Kf, Fin, dhW, W, dH);
    mm_nt(V, (u64)r, Fin, dpl, Pl, t.data());
    for (u64 i = 0; i < V * Fin; ++i) dH[i] += t[i];
    mm_nt(V, (u64)r, Fin, dpr, Pr, t.data());
    for (u64 i = 0; i < V * Fin; ++i) dH[i] += t[i];
  }
}

// ---------------------------------------------------------------------------
// GCN (PAPER.md:534-540 ): h'_v = sigma(b + sum_{(u,e,v)} w_e h_u W).
// The weighted Aggregate over one index (csr_dst forward; csc_src = the transpose in
// backward), edge weights looked up by edge id -- the same per-row sum as
// dense_aggregate but walked in index order.
// ---------------------------------------------------------------------------
}  // extern "C"

template <typename T>
static void gcn_aggregate(u64 R, const u64* off, const u32* nbr, const u32* eid, const T* w, int F, const T* X,
                          const T* bias, int relu, T* Y) {
#pragma omp parallel for schedule(dynamic, 64) if (R > 4096)
  for (long long r = 0; r < (long long)R; ++r) {
    T* y = Y + (u64)r * F;
    for (int j = 0; j < F; ++j) y[j] = 0;
    for (u64 i = off[r]; i < off[r + 1]; ++i) {
      const T a = w ? w[eid[i]] : T(1);
      const T* x = X + (u64)nbr[i] * F;
      for (int j = 0; j < F; ++j) y[j] += a * x[j];
    }
    for (int j = 0; j < F; ++j) {
      const T z = y[j] + (bias ? bias[j] : T(0));
      y[j] = (relu && !(z > 0)) ? T(0) : z;
    }
  }
}

extern "C" {

void orc_gcn_aggregate_f64(u64 R, const u64* off, const u32* nbr, const u32* eid, const double* w, int F,
                           const double* X, const double* bias, int relu, double* Y) {
  gcn_aggregate(R, off, nbr, eid, w, F, X, bias, relu, Y);
}
void orc_gcn_aggregate_f32(u64 R, const u64* off, const u32* nbr, const u32* eid, const float* w, int F,
                           const float* X, const float* bias, int relu, float* Y) {
  gcn_aggregate(R, off, nbr, eid, w, F, X, bias, relu, Y);
}

// Symmetric normalisation w_e = 1/sqrt(max(1,deg_in(dst)) max(1,deg_out(src))).
void orc_gcn_norm(u64 V, u64 E, const u32* src, const u32* dst, const u64* doff, const u64* soff, float* w) {
  (void)V;
  for (u64 e = 0; e < E; ++e) {
    const double din = (double)std::max<u64>(1, doff[dst[e] + 1] - doff[dst[e]]);
    const double dout = (double)std::max<u64>(1, soff[src[e] + 1] - soff[src[e]]);
    w[e] = (float)(1.0 / std::sqrt(din * dout));
  }
}

// ---------------------------------------------------------------------------
// Cost-algebra closed forms (SPEC.md:282-289 ), element
// counts.  Used as known-answer checks (G3: 39 -> 30 flops, 45 -> 33 IO units).
// ---------------------------------------------------------------------------
u64 orc_gat_attn_flops_naive(u64 V, u64 E, u64 f) { (void)V; return 6 * E * f + E; }
u64 orc_gat_attn_flops_reorg(u64 V, u64 E, u64 f) { return 4 * V * f + 2 * E; }
u64 orc_gat_io_unfused(u64 V, u64 E, u64 h, u64 f) { return V * h * f + 7 * E * h + 3 * E * h * f; }
u64 orc_gat_io_fused(u64 V, u64 E, u64 h, u64 f) { return V * h * f + 5 * E * h + 2 * E * h * f; }

// ---------------------------------------------------------------------------
// Chung-Lu generator restated on the host (OpenMP): the same counter-based draws as the
// device's gnncg_gen_chung_lu and graph.py:chung_lu_edges_host (test / CPU-arm input
// only; the full C2 graph for bench.py --impl reference).
// ---------------------------------------------------------------------------
static inline u64 orc_splitmix64(u64 x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static inline u32 orc_sample_cdf(const u64* cdf, u64 V, u64 r) {
  // smallest i with cdf[i] > r
  return (u32)(std::upper_bound(cdf, cdf + V, r) - cdf);
}

void orc_gen_chung_lu(u64 V, u64 E, const u64* cdf, u64 seed, u32* src, u32* dst) {
  const u64 total = cdf[V - 1];
#pragma omp parallel for schedule(static)
  for (i64 ee = 0; ee < (i64)E; ++ee) {
    const u64 e = (u64)ee;
    const u64 h0 = orc_splitmix64(seed * 0xD1B54A32D192ED03ull + 2ull * e);
    const u64 h1 = orc_splitmix64(seed * 0xD1B54A32D192ED03ull + 2ull * e + 1ull);
    dst[e] = orc_sample_cdf(cdf, V, (u64)(((unsigned __int128)h0 * total) >> 64));
    src[e] = orc_sample_cdf(cdf, V, (u64)(((unsigned __int128)h1 * total) >> 64));
  }
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

}  // extern "C"
