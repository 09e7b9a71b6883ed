// SPDX-License-Identifier: Apache-2.0
//
// gnncg_b200/ops.hpp -- header-only C++ operator API of the B200 fused GNN layer path,
// written against the reference's own types (gnncg::Graph, graph.hpp:34-65;
// gnncg::Tensor<float>, tensor.hpp:20-35) and error classes (GraphError,
// TensorError).  It is what a reference executor (run_forward /
// run_backward / train_step) calls in place of its CPU fused regions:
//
//   b200::DeviceGraph dg(graph);                          // upload + device CSR/CSC (bit-exact)
//   b200::GatStash st;
//   Tensor<float> out = b200::gat_forward(dg, H, W, a_l, a_r, {8, 32}, &st);
//   b200::GatGrads gr = b200::gat_backward(dg, H, W, a_l, a_r, st, dOut, {8, 32}, true);
//
// Host tensors in, host tensors out (copies on the graph's stream); the device
// stash stays resident between forward and backward.  Every FLOP runs in
// libgnncg_b200.so through the C ABI of gnncg_b200.h; there is no CPU fallback.
// Include after <gnncg/graph.hpp> and <gnncg/tensor.hpp>.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>  // tensor.hpp uses std::max(initializer_list) without including these
#include <cstdint>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gnncg/graph.hpp"
#include "gnncg/tensor.hpp"
#include "gnncg_b200.h"

namespace gnncg {
namespace b200 {

// Map a C-ABI status to the reference's exception types.
inline void check(int rc, const char* what) {
  if (rc == GNNCG_OK) return;
  const std::string msg = std::string(what) + ": " + gnncg_last_error();
  if (rc == GNNCG_ERR_SHAPE) throw TensorError(msg);
  if (rc == GNNCG_ERR_RANGE) throw GraphError(msg);
  throw std::runtime_error(msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Owning device allocation.
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t bytes) : bytes_(bytes) {
    if (bytes) cuda_check(cudaMalloc(&ptr_, bytes), "cudaMalloc");
  }
  DeviceBuffer(DeviceBuffer&& o) noexcept : ptr_(o.ptr_), bytes_(o.bytes_) { o.ptr_ = nullptr; o.bytes_ = 0; }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(ptr_, o.ptr_);
    std::swap(bytes_, o.bytes_);
    return *this;
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() { if (ptr_) cudaFree(ptr_); }
  template <typename T = void>
  T* get() const { return static_cast<T*>(ptr_); }
  size_t bytes() const { return bytes_; }
  void ensure(size_t bytes) { if (bytes > bytes_) *this = DeviceBuffer(bytes); }

 private:
  void* ptr_ = nullptr;
  size_t bytes_ = 0;
};

template <typename T>
DeviceBuffer upload(const T* host, size_t n, cudaStream_t s) {
  DeviceBuffer b(n * sizeof(T));
  if (n) cuda_check(cudaMemcpyAsync(b.get(), host, n * sizeof(T), cudaMemcpyHostToDevice, s), "upload");
  return b;
}

inline DeviceBuffer upload(const Tensor<float>& t, cudaStream_t s) { return upload(t.data.data(), t.size(), s); }

inline Tensor<float> download(const DeviceBuffer& b, std::uint64_t rows, std::uint64_t cols, cudaStream_t s) {
  Tensor<float> t(rows, cols);
  if (t.size()) {
    cuda_check(cudaMemcpyAsync(t.data.data(), b.get(), t.size() * sizeof(float), cudaMemcpyDeviceToHost, s),
               "download");
    cuda_check(cudaStreamSynchronize(s), "sync");
  }
  return t;
}

// One adjacency index in HBM plus its edge-balance schedule.
struct DeviceIndex {
  std::int64_t rows = 0, edges = 0;
  DeviceBuffer off, nbr, eid;
  DeviceBuffer items, split_rows, split_first;
  std::vector<std::uint64_t> host_off;  // host copy of off (the other index's L2 gather hint)
  gnncg_sched_t sched{};

  gnncg_index_t view() const {
    return gnncg_index_t{rows, edges, off.get<std::uint64_t>(), nbr.get<std::uint32_t>(), eid.get<std::uint32_t>()};
  }
};

// gnncg::Graph resident in HBM: both indexes rebuilt on the device by the
// bit-exact counting sort (gnncg_csr_build == build_index, graph.cpp:14-28).
class DeviceGraph {
 public:
  explicit DeviceGraph(const Graph& g, std::int32_t chunk = 2048, cudaStream_t stream = nullptr)
      : V_(static_cast<std::int64_t>(g.num_vertices())), E_(static_cast<std::int64_t>(g.num_edges())), s_(stream) {
    check(gnncg_device_check(), "gnncg_device_check");
    std::vector<std::uint32_t> src(E_), dst(E_);
    for (std::int64_t e = 0; e < E_; ++e) {
      src[e] = g.edge_src(static_cast<EdgeId>(e));
      dst[e] = g.edge_dst(static_cast<EdgeId>(e));
    }
    edge_src_ = upload(src.data(), src.size(), s_);
    edge_dst_ = upload(dst.data(), dst.size(), s_);
    DeviceBuffer ws(gnncg_csr_build_workspace(V_, E_));
    build(dst_, edge_dst_, edge_src_, ws, chunk);
    build(src_, edge_src_, edge_dst_, ws, chunk);
    // L2 hint (gnncg_l2_persist): K2 over csr_dst gathers source rows, read out-degree times;
    // K4f over csc_src gathers destination rows, read in-degree times
    dst_.sched.gather_off = src_.host_off.data();
    dst_.sched.gather_rows = V_;
    src_.sched.gather_off = dst_.host_off.data();
    src_.sched.gather_rows = V_;
  }

  std::int64_t num_vertices() const { return V_; }
  std::int64_t num_edges() const { return E_; }
  const DeviceIndex& csr_dst() const { return dst_; }
  const DeviceIndex& csc_src() const { return src_; }
  const std::uint32_t* edge_src() const { return edge_src_.get<std::uint32_t>(); }
  const std::uint32_t* edge_dst() const { return edge_dst_.get<std::uint32_t>(); }
  cudaStream_t stream() const { return s_; }
  DeviceBuffer& workspace(size_t bytes) const {
    ws_.ensure(bytes);
    return ws_;
  }

 private:
  void build(DeviceIndex& idx, const DeviceBuffer& key, const DeviceBuffer& other, DeviceBuffer& ws,
             std::int32_t chunk) {
    build_index(idx, V_, V_, E_, key.get<std::uint32_t>(), other.get<std::uint32_t>(), ws, chunk, s_);
  }

 public:
  // One index of `rows` rows over neighbour ids [0, n_other) from device key / other arrays
  // (gnncg_csr_build_rect: the reference's counting sort, stable in edge id) plus its schedule.
  static void build_index(DeviceIndex& idx, std::int64_t rows, std::int64_t n_other, std::int64_t E,
                          const std::uint32_t* key, const std::uint32_t* other, DeviceBuffer& ws, std::int32_t chunk,
                          cudaStream_t s) {
    ws.ensure(gnncg_csr_build_workspace(rows, E));
    idx.rows = rows;
    idx.edges = E;
    idx.off = DeviceBuffer((rows + 1) * sizeof(std::uint64_t));
    idx.nbr = DeviceBuffer(std::max<std::int64_t>(E, 1) * sizeof(std::uint32_t));
    idx.eid = DeviceBuffer(std::max<std::int64_t>(E, 1) * sizeof(std::uint32_t));
    check(gnncg_csr_build_rect(rows, n_other, E, key, other, idx.off.get<std::uint64_t>(), idx.nbr.get<std::uint32_t>(),
                               idx.eid.get<std::uint32_t>(), ws.get(), ws.bytes(), s),
          "gnncg_csr_build_rect");
    std::vector<std::uint64_t> off(rows + 1);
    cuda_check(cudaMemcpyAsync(off.data(), idx.off.get(), off.size() * 8, cudaMemcpyDeviceToHost, s), "offsets");
    cuda_check(cudaStreamSynchronize(s), "sync");
    std::int64_t n = 0, ns = 0, nr = 0;
    check(gnncg_sched_build_host(rows, off.data(), chunk, &n, &ns, &nr, nullptr, nullptr, nullptr), "sched");
    std::vector<std::uint32_t> items(2 * n + 2), srows(nr + 1), first(nr + 1);
    check(gnncg_sched_build_host(rows, off.data(), chunk, &n, &ns, &nr, items.data(), srows.data(), first.data()),
          "sched");
    idx.host_off = std::move(off);
    idx.items = upload(items.data(), items.size(), s);
    idx.split_rows = upload(srows.data(), srows.size(), s);
    idx.split_first = upload(first.data(), first.size(), s);
    idx.sched = gnncg_sched_t{n, ns, nr, chunk, 0, idx.items.get<std::uint32_t>(), idx.split_rows.get<std::uint32_t>(),
                              idx.split_first.get<std::uint32_t>()};
  }

 private:
  std::int64_t V_, E_;
  cudaStream_t s_;
  DeviceBuffer edge_src_, edge_dst_;
  DeviceIndex dst_, src_;
  mutable DeviceBuffer ws_;
};

// Gather tables of the fused kernels: fp32 (the 1e-4 contract) or bf16 (Ht / dOut rows read
// from bf16 copies, all arithmetic fp32; the north star's "bf16 features" option with a looser
// bound, see gnncg_gat_fwd_bf16).
enum class Gather { fp32, bf16 };
// Backward: deterministic = K3 (csr_dst) + K4 (csc_src), fixed-order, bitwise reproducible;
// fast = one fused csc_src pass with dA_r by global reductions (SPEC.md:378 fast mode).
enum class Backward { deterministic, fast };

struct GatParams {
  int heads;
  int f;
  float slope = 0.2f;  // tensor.hpp:93
  Gather gather = Gather::fp32;
  Backward backward = Backward::deterministic;  // bf16 gather always uses the fast backward
};

// O(|V|) forward state kept for the backward, plus the layer output (the fast
// backward's row dot) and the bf16 gather copy of Ht when gather == bf16.
struct GatStash {
  DeviceBuffer Ht, Al, Ar, m, d, out, Ht_lp;
};

struct GatGrads {
  Tensor<float> dH, dW, da_l, da_r;
};

// Opt in to L2-persisting windows over the hottest gathered rows of the fused GAT kernels
// (gnncg_l2_persist; DeviceGraph's schedules carry the hint).  Returns the set-aside granted.
inline size_t l2_persist(size_t bytes) {
  size_t got = 0;
  check(gnncg_l2_persist(bytes, &got), "gnncg_l2_persist");
  return got;
}

namespace detail {

inline void require_shape(const Tensor<float>& t, std::uint64_t r, std::uint64_t c, const char* name) {
  if (t.rows != r || t.cols != c)
    throw TensorError(std::string(name) + ": shape mismatch (" + std::to_string(t.rows) + "x" +
                      std::to_string(t.cols) + " vs " + std::to_string(r) + "x" + std::to_string(c) + ")");
}

inline void gemm(const DeviceGraph& g, int ta, int tb, std::int64_t M, std::int64_t N, std::int64_t K, const float* A,
                 std::int64_t lda, const float* B, std::int64_t ldb, float* C, std::int64_t ldc) {
  DeviceBuffer& ws = g.workspace(gnncg_gemm_workspace(ta, tb, M, N, K));
  check(gnncg_gemm(ta, tb, M, N, K, A, lda, B, ldb, C, ldc, ws.get(), ws.bytes(), g.stream()), "gnncg_gemm");
}
}  // namespace detail

// GAT layer forward, reorganized and fused.
inline Tensor<float> gat_forward(const DeviceGraph& g, const Tensor<float>& H, const Tensor<float>& W,
                                 const Tensor<float>& a_l, const Tensor<float>& a_r, const GatParams& p,
                                 GatStash* stash) {
  const std::int64_t V = g.num_vertices(), h = p.heads, f = p.f, hf = h * f;
  detail::require_shape(H, V, H.cols, "gat_forward H");
  detail::require_shape(W, H.cols, hf, "gat_forward W");
  detail::require_shape(a_l, h, f, "gat_forward a_l");
  detail::require_shape(a_r, h, f, "gat_forward a_r");
  cudaStream_t s = g.stream();
  GatStash local;
  GatStash& st = stash ? *stash : local;
  DeviceBuffer dH = upload(H, s), dW = upload(W, s), dal = upload(a_l, s), dar = upload(a_r, s);
  st.Ht = DeviceBuffer(V * hf * 4);
  st.Al = DeviceBuffer(V * h * 4);
  st.Ar = DeviceBuffer(V * h * 4);
  st.m = DeviceBuffer(V * h * 4);
  st.d = DeviceBuffer(V * h * 4);
  {  // K1 with the attention-LP epilogue (one tensor-core GEMM)
    DeviceBuffer& gws = g.workspace(gnncg_gemm_workspace(0, 0, V, hf, H.cols));
    check(gnncg_gat_transform(V, H.cols, h, f, dH.get<float>(), H.cols, dW.get<float>(), st.Ht.get<float>(),
                              dal.get<float>(), dar.get<float>(), st.Al.get<float>(), st.Ar.get<float>(), gws.get(),
                              gws.bytes(), s),
          "gnncg_gat_transform");
  }
  st.out = DeviceBuffer(V * hf * 4);
  const gnncg_index_t idx = g.csr_dst().view();
  DeviceBuffer& ws = g.workspace(gnncg_gat_workspace(&g.csr_dst().sched, nullptr, h, f));
  if (p.gather == Gather::bf16) {
    if (!gnncg_gat_bf16_supported(p.heads, p.f)) throw TensorError("gat_forward: bf16 gather unsupported for this shape");
    st.Ht_lp = DeviceBuffer(V * hf * 2);
    check(gnncg_pack_bf16(V * hf, st.Ht.get<float>(), st.Ht_lp.get<std::uint16_t>(), s), "gnncg_pack_bf16");
    check(gnncg_gat_fwd_bf16(&idx, &g.csr_dst().sched, h, f, p.slope, st.Ht_lp.get<std::uint16_t>(),
                             st.Al.get<float>(), st.Ar.get<float>(), st.out.get<float>(), st.m.get<float>(),
                             st.d.get<float>(), ws.get(), ws.bytes(), s),
          "gnncg_gat_fwd_bf16");
  } else {
    check(gnncg_gat_fwd(&idx, &g.csr_dst().sched, h, f, p.slope, st.Ht.get<float>(), st.Al.get<float>(),
                        st.Ar.get<float>(), st.out.get<float>(), st.m.get<float>(), st.d.get<float>(), ws.get(),
                        ws.bytes(), s),
          "gnncg_gat_fwd");
  }
  return download(st.out, V, hf, s);
}

// GAT layer backward with recomputation.
inline GatGrads gat_backward(const DeviceGraph& g, const Tensor<float>& H, const Tensor<float>& W,
                             const Tensor<float>& a_l, const Tensor<float>& a_r, const GatStash& st,
                             const Tensor<float>& dOut, const GatParams& p, bool need_dH) {
  const std::int64_t V = g.num_vertices(), h = p.heads, f = p.f, hf = h * f, Fin = H.cols;
  detail::require_shape(dOut, V, hf, "gat_backward dOut");
  detail::require_shape(W, Fin, hf, "gat_backward W");
  cudaStream_t s = g.stream();
  DeviceBuffer dH_in = upload(H, s), dW_in = upload(W, s), dal_in = upload(a_l, s), dar_in = upload(a_r, s);
  DeviceBuffer g_out = upload(dOut, s);
  DeviceBuffer c(V * h * 4), dAr(V * h * 4), dAl(V * h * 4), dHt(V * hf * 4), da_l(hf * 4), da_r(hf * 4);
  const gnncg_index_t csr = g.csr_dst().view(), csc = g.csc_src().view();
  size_t need = gnncg_gat_workspace(&g.csr_dst().sched, &g.csc_src().sched, h, f);
  need = std::max(need, gnncg_gat_attn_grad_workspace(V, h, f));
  DeviceBuffer& ws = g.workspace(need);
  const bool lp = p.gather == Gather::bf16;
  if (lp || p.backward == Backward::fast) {
    if (!lp && !gnncg_gat_fast_supported(p.heads, p.f)) throw TensorError("gat_backward: fast mode unsupported here");
    DeviceBuffer rec(V * gnncg_gat_rec_stride(p.heads) * 4);
    if (lp) {
      DeviceBuffer g_lp(V * hf * 2);
      check(gnncg_gat_bwd_prep_bf16(V, h, f, g_out.get<float>(), st.out.get<float>(), st.Ar.get<float>(),
                                    st.m.get<float>(), st.d.get<float>(), rec.get<float>(),
                                    g_lp.get<std::uint16_t>(), s),
            "gnncg_gat_bwd_prep_bf16");
      check(gnncg_gat_bwd_src_fused_bf16(&csc, &g.csc_src().sched, h, f, p.slope, 0, V,
                                         st.Ht_lp.get<std::uint16_t>(), st.Al.get<float>(), rec.get<float>(),
                                         g_lp.get<std::uint16_t>(), dal_in.get<float>(), dar_in.get<float>(),
                                         dHt.get<float>(), dAl.get<float>(), dAr.get<float>(), ws.get(), ws.bytes(), s),
            "gnncg_gat_bwd_src_fused_bf16");
      cuda_check(cudaStreamSynchronize(s), "sync");  // g_lp / rec are released at scope end
    } else {
      check(gnncg_gat_bwd_prep(V, h, f, g_out.get<float>(), st.out.get<float>(), st.Ar.get<float>(), st.m.get<float>(),
                               st.d.get<float>(), rec.get<float>(), s),
            "gnncg_gat_bwd_prep");
      check(gnncg_gat_bwd_src_fused(&csc, &g.csc_src().sched, h, f, p.slope, 0, V, st.Ht.get<float>(),
                                    st.Al.get<float>(), rec.get<float>(), g_out.get<float>(), dal_in.get<float>(),
                                    dar_in.get<float>(), dHt.get<float>(), dAl.get<float>(), dAr.get<float>(), ws.get(),
                                    ws.bytes(), s),
            "gnncg_gat_bwd_src_fused");
      cuda_check(cudaStreamSynchronize(s), "sync");
    }
  } else {
    check(gnncg_gat_bwd_dst(&csr, &g.csr_dst().sched, h, f, p.slope, st.Ht.get<float>(), st.Al.get<float>(),
                            st.Ar.get<float>(), st.m.get<float>(), st.d.get<float>(), g_out.get<float>(),
                            c.get<float>(), dAr.get<float>(), ws.get(), ws.bytes(), s),
          "gnncg_gat_bwd_dst");
    check(gnncg_gat_bwd_src(&csc, &g.csc_src().sched, h, f, p.slope, 0, V, st.Ht.get<float>(), st.Al.get<float>(),
                            st.Ar.get<float>(), st.m.get<float>(), st.d.get<float>(), c.get<float>(),
                            g_out.get<float>(), dAr.get<float>(), dal_in.get<float>(), dar_in.get<float>(),
                            dHt.get<float>(), dAl.get<float>(), ws.get(), ws.bytes(), s),
          "gnncg_gat_bwd_src");
  }
  check(gnncg_gat_attn_grad(V, h, f, st.Ht.get<float>(), dAl.get<float>(), dAr.get<float>(), da_l.get<float>(),
                            da_r.get<float>(), ws.get(), ws.bytes(), s),
        "gnncg_gat_attn_grad");
  GatGrads out;
  DeviceBuffer dW(Fin * hf * 4);
  detail::gemm(g, 1, 0, Fin, hf, V, dH_in.get<float>(), Fin, dHt.get<float>(), hf, dW.get<float>(), hf);
  out.dW = download(dW, Fin, hf, s);
  out.da_l = download(da_l, h, f, s);
  out.da_r = download(da_r, h, f, s);
  if (need_dH) {
    DeviceBuffer dHb(V * Fin * 4);
    detail::gemm(g, 0, 1, V, Fin, hf, dHt.get<float>(), hf, dW_in.get<float>(), hf, dHb.get<float>(), Fin);
    out.dH = download(dHb, V, Fin, s);
  }
  return out;
}

// EdgeConv layer forward: returns out; argmax (edge ids) via *argmax.
inline Tensor<float> edgeconv_forward(const DeviceGraph& g, const Tensor<float>& H, const Tensor<float>& Theta,
                                      const Tensor<float>& Phi, std::vector<std::uint32_t>* argmax) {
  const std::int64_t V = g.num_vertices(), Fin = H.cols, C = Theta.cols;
  detail::require_shape(Theta, Fin, C, "edgeconv Theta");
  detail::require_shape(Phi, Fin, C, "edgeconv Phi");
  cudaStream_t s = g.stream();
  Tensor<float> Wc(Fin, 2 * C);
  for (std::int64_t i = 0; i < Fin; ++i)
    for (std::int64_t c = 0; c < C; ++c) {
      Wc.at(i, c) = Theta.at(i, c);
      Wc.at(i, C + c) = Phi.at(i, c);
    }
  DeviceBuffer dH = upload(H, s), dWc = upload(Wc, s), Y(V * 2 * C * 4), out(V * C * 4), am(V * C * 4);
  detail::gemm(g, 0, 0, V, 2 * C, Fin, dH.get<float>(), Fin, dWc.get<float>(), 2 * C, Y.get<float>(), 2 * C);
  const gnncg_index_t csr = g.csr_dst().view();
  check(gnncg_edgeconv_fwd(&csr, (int)C, 0, Y.get<float>(), 2 * C, Y.get<float>() + C, 2 * C, out.get<float>(),
                           am.get<std::uint32_t>(), s),
        "gnncg_edgeconv_fwd");
  if (argmax) {
    argmax->resize(V * C);
    cuda_check(cudaMemcpyAsync(argmax->data(), am.get(), V * C * 4, cudaMemcpyDeviceToHost, s), "argmax");
  }
  return download(out, V, C, s);
}

struct EdgeConvGrads {
  Tensor<float> dH, dTheta, dPhi;
};

// EdgeConv backward: argmax routing then the two backward Applies.
// `argmax` is the edge-id tensor returned by edgeconv_forward.
inline EdgeConvGrads edgeconv_backward(const DeviceGraph& g, const Tensor<float>& H, const Tensor<float>& Theta,
                                       const Tensor<float>& Phi, const std::vector<std::uint32_t>& argmax,
                                       const Tensor<float>& dOut, bool need_dH) {
  const std::int64_t V = g.num_vertices(), Fin = H.cols, C = Theta.cols;
  detail::require_shape(dOut, V, C, "edgeconv_backward dOut");
  if ((std::int64_t)argmax.size() != V * C) throw TensorError("edgeconv_backward: argmax size != V*C");
  cudaStream_t s = g.stream();
  Tensor<float> Wc(Fin, 2 * C);
  for (std::int64_t i = 0; i < Fin; ++i)
    for (std::int64_t c = 0; c < C; ++c) {
      Wc.at(i, c) = Theta.at(i, c);
      Wc.at(i, C + c) = Phi.at(i, c);
    }
  DeviceBuffer dH = upload(H, s), dWc = upload(Wc, s), g_out = upload(dOut, s);
  DeviceBuffer am = upload(argmax.data(), argmax.size(), s), dY(V * 2 * C * 4), dW(Fin * 2 * C * 4);
  const gnncg_index_t csr = g.csr_dst().view(), csc = g.csc_src().view();
  check(gnncg_edgeconv_bwd(&csc, &csr, (int)C, am.get<std::uint32_t>(), g_out.get<float>(), dY.get<float>(), 2 * C,
                           dY.get<float>() + C, 2 * C, s),
        "gnncg_edgeconv_bwd");
  detail::gemm(g, 1, 0, Fin, 2 * C, V, dH.get<float>(), Fin, dY.get<float>(), 2 * C, dW.get<float>(), 2 * C);
  EdgeConvGrads out;
  const Tensor<float> dWh = download(dW, Fin, 2 * C, s);
  out.dTheta = Tensor<float>(Fin, C);
  out.dPhi = Tensor<float>(Fin, C);
  for (std::int64_t i = 0; i < Fin; ++i)
    for (std::int64_t c = 0; c < C; ++c) {
      out.dTheta.at(i, c) = dWh.at(i, c);
      out.dPhi.at(i, c) = dWh.at(i, C + c);
    }
  if (need_dH) {
    DeviceBuffer dHb(V * Fin * 4);
    detail::gemm(g, 0, 1, V, Fin, 2 * C, dY.get<float>(), 2 * C, dWc.get<float>(), 2 * C, dHb.get<float>(), Fin);
    out.dH = download(dHb, V, Fin, s);
  }
  return out;
}

// GMMConv: parameters W (F_in x K*f), P_l, P_r (F_in x r), mu, sinv (K x r).
struct GmmParams {
  int K, r, f;
};

struct GmmStash {
  DeviceBuffer Y;  // [hW | pl | pr], V x (K f + 2 r)
  std::int64_t ldy = 0;
};

struct GmmGrads {
  Tensor<float> dH, dW, dP_l, dP_r, dmu, dsinv;
};

namespace detail {
// [parts...] side by side; ld > the total width pads with zero columns (16-byte rows for the
// tensor-core GEMM)
inline Tensor<float> pack_cols(const std::vector<const Tensor<float>*>& parts, std::uint64_t ld = 0) {
  std::uint64_t cols = 0;
  for (auto* p : parts) cols += p->cols;
  Tensor<float> out(parts[0]->rows, std::max(cols, ld), 0.0f);
  std::uint64_t c0 = 0;
  for (auto* p : parts) {
    for (std::uint64_t i = 0; i < p->rows; ++i)
      for (std::uint64_t c = 0; c < p->cols; ++c) out.at(i, c0 + c) = p->at(i, c);
    c0 += p->cols;
  }
  return out;
}
}  // namespace detail

inline Tensor<float> gmm_forward(const DeviceGraph& g, const Tensor<float>& H, const Tensor<float>& W,
                                 const Tensor<float>& P_l, const Tensor<float>& P_r, const Tensor<float>& mu,
                                 const Tensor<float>& sinv, const GmmParams& p, GmmStash* stash) {
  const std::int64_t V = g.num_vertices(), Fin = H.cols, Kf = (std::int64_t)p.K * p.f;
  const std::int64_t ldy = (Kf + 2 * p.r + 3) / 4 * 4;  // zero-padded to 16-byte rows
  detail::require_shape(W, Fin, Kf, "gmm W");
  detail::require_shape(P_l, Fin, p.r, "gmm P_l");
  detail::require_shape(P_r, Fin, p.r, "gmm P_r");
  detail::require_shape(mu, p.K, p.r, "gmm mu");
  detail::require_shape(sinv, p.K, p.r, "gmm sinv");
  cudaStream_t s = g.stream();
  GmmStash local;
  GmmStash& st = stash ? *stash : local;
  DeviceBuffer dH = upload(H, s), dWc = upload(detail::pack_cols({&W, &P_l, &P_r}, ldy), s);
  DeviceBuffer dmu = upload(mu, s), dsi = upload(sinv, s), out(V * p.f * 4);
  st.Y = DeviceBuffer(V * ldy * 4);
  st.ldy = ldy;
  detail::gemm(g, 0, 0, V, ldy, Fin, dH.get<float>(), Fin, dWc.get<float>(), ldy, st.Y.get<float>(), ldy);
  const gnncg_index_t csr = g.csr_dst().view();
  check(gnncg_gmm_fwd(&csr, p.K, p.r, p.f, st.Y.get<float>(), ldy, dmu.get<float>(), dsi.get<float>(),
                      out.get<float>(), s),
        "gnncg_gmm_fwd");
  return download(out, V, p.f, s);
}

inline GmmGrads gmm_backward(const DeviceGraph& g, const Tensor<float>& H, const Tensor<float>& W,
                             const Tensor<float>& P_l, const Tensor<float>& P_r, const Tensor<float>& mu,
                             const Tensor<float>& sinv, const GmmParams& p, const GmmStash& st,
                             const Tensor<float>& dOut, bool need_dH) {
  const std::int64_t V = g.num_vertices(), Fin = H.cols, Kf = (std::int64_t)p.K * p.f, ldy = st.ldy;
  detail::require_shape(dOut, V, p.f, "gmm dOut");
  cudaStream_t s = g.stream();
  DeviceBuffer dH = upload(H, s), dWc = upload(detail::pack_cols({&W, &P_l, &P_r}, ldy), s);
  DeviceBuffer dmu_in = upload(mu, s), dsi_in = upload(sinv, s), g_out = upload(dOut, s);
  DeviceBuffer dY(V * ldy * 4), dmu(p.K * p.r * 4), dsinv(p.K * p.r * 4), dW(Fin * ldy * 4);
  if (V > 0) cuda_check(cudaMemsetAsync(dY.get(), 0, dY.bytes(), s), "memset dY");  // K8 leaves the padding
  const gnncg_index_t csr = g.csr_dst().view(), csc = g.csc_src().view();
  DeviceBuffer& ws = g.workspace(gnncg_gmm_bwd_workspace(&csr, p.K, p.r));
  check(gnncg_gmm_bwd(&csr, &csc, p.K, p.r, p.f, st.Y.get<float>(), ldy, dmu_in.get<float>(), dsi_in.get<float>(),
                      g_out.get<float>(), dY.get<float>(), dmu.get<float>(), dsinv.get<float>(), ws.get(), ws.bytes(),
                      s),
        "gnncg_gmm_bwd");
  detail::gemm(g, 1, 0, Fin, ldy, V, dH.get<float>(), Fin, dY.get<float>(), ldy, dW.get<float>(), ldy);
  GmmGrads out;
  const Tensor<float> dWh = download(dW, Fin, ldy, s);
  out.dW = Tensor<float>(Fin, Kf);
  out.dP_l = Tensor<float>(Fin, p.r);
  out.dP_r = Tensor<float>(Fin, p.r);
  for (std::int64_t i = 0; i < Fin; ++i) {
    for (std::int64_t c = 0; c < Kf; ++c) out.dW.at(i, c) = dWh.at(i, c);
    for (std::int64_t c = 0; c < p.r; ++c) {
      out.dP_l.at(i, c) = dWh.at(i, Kf + c);
      out.dP_r.at(i, c) = dWh.at(i, Kf + p.r + c);
    }
  }
  out.dmu = download(dmu, p.K, p.r, s);
  out.dsinv = download(dsinv, p.K, p.r, s);
  if (need_dH) {
    DeviceBuffer dHb(V * Fin * 4);
    detail::gemm(g, 0, 1, V, Fin, ldy, dY.get<float>(), ldy, dWc.get<float>(), ldy, dHb.get<float>(), Fin);
    out.dH = download(dHb, V, Fin, s);
  }
  return out;
}

// GCN: out = relu(b + sum_e w_e H[u] W) with the symmetric
// normalisation w_e = 1/sqrt(max(1,deg_in(v)) max(1,deg_out(u))) computed on the device.
struct GcnStash {
  DeviceBuffer Ht, out, w;
};

struct GcnGrads {
  Tensor<float> dH, dW, db;
};

inline Tensor<float> gcn_forward(const DeviceGraph& g, const Tensor<float>& H, const Tensor<float>& W,
                                 const Tensor<float>& b, GcnStash* stash) {
  const std::int64_t V = g.num_vertices(), Fin = H.cols, C = W.cols;
  detail::require_shape(W, Fin, C, "gcn W");
  detail::require_shape(b, 1, C, "gcn b");
  cudaStream_t s = g.stream();
  GcnStash local;
  GcnStash& st = stash ? *stash : local;
  DeviceBuffer dH = upload(H, s), dW = upload(W, s), db = upload(b, s);
  st.Ht = DeviceBuffer(V * C * 4);
  st.out = DeviceBuffer(V * C * 4);
  st.w = DeviceBuffer(g.num_edges() * 4);
  const gnncg_index_t csr = g.csr_dst().view(), csc = g.csc_src().view();
  check(gnncg_gcn_norm(g.num_edges(), g.edge_src(), g.edge_dst(), &csr, &csc, st.w.get<float>(), s), "gnncg_gcn_norm");
  detail::gemm(g, 0, 0, V, C, Fin, dH.get<float>(), Fin, dW.get<float>(), C, st.Ht.get<float>(), C);
  DeviceBuffer& ws = g.workspace(gnncg_spmm_workspace(&g.csr_dst().sched, (int)C));
  check(gnncg_spmm(&csr, &g.csr_dst().sched, (int)C, st.w.get<float>(), st.Ht.get<float>(), db.get<float>(), 1,
                   st.out.get<float>(), ws.get(), ws.bytes(), s),
        "gnncg_spmm");
  return download(st.out, V, C, s);
}

inline GcnGrads gcn_backward(const DeviceGraph& g, const Tensor<float>& H, const Tensor<float>& W, const GcnStash& st,
                             const Tensor<float>& dOut, bool need_dH) {
  const std::int64_t V = g.num_vertices(), Fin = H.cols, C = W.cols;
  detail::require_shape(dOut, V, C, "gcn dOut");
  cudaStream_t s = g.stream();
  DeviceBuffer dH = upload(H, s), dWin = upload(W, s), g_out = upload(dOut, s);
  DeviceBuffer dZ(V * C * 4), db(C * 4), dHt(V * C * 4), dW(Fin * C * 4);
  {
    DeviceBuffer& ws = g.workspace(gnncg_relu_bwd_workspace((int)C));
    check(gnncg_relu_bwd(V, (int)C, g_out.get<float>(), st.out.get<float>(), 1, dZ.get<float>(), db.get<float>(),
                         ws.get(), ws.bytes(), s),
          "gnncg_relu_bwd");
  }
  const gnncg_index_t csc = g.csc_src().view();
  DeviceBuffer& ws = g.workspace(gnncg_spmm_workspace(&g.csc_src().sched, (int)C));
  check(gnncg_spmm(&csc, &g.csc_src().sched, (int)C, st.w.get<float>(), dZ.get<float>(), nullptr, 0, dHt.get<float>(),
                   ws.get(), ws.bytes(), s),
        "gnncg_spmm");
  detail::gemm(g, 1, 0, Fin, C, V, dH.get<float>(), Fin, dHt.get<float>(), C, dW.get<float>(), C);
  GcnGrads out;
  out.dW = download(dW, Fin, C, s);
  out.db = download(db, 1, C, s);
  if (need_dH) {
    DeviceBuffer dHb(V * Fin * 4);
    detail::gemm(g, 0, 1, V, Fin, C, dHt.get<float>(), C, dWin.get<float>(), C, dHb.get<float>(), Fin);
    out.dH = download(dHb, V, Fin, s);
  }
  return out;
}

// ------------------------------------------------------------------ multi-GPU
// One process per GPU, destination rows partitioned over the ranks (north_star).
// A reference executor running P ranks calls these in place of its run_forward / run_backward
// for the rank's rows; the collectives run inside the library
// (gnncg_gat_fwd_dist / gnncg_gat_bwd_dist) over a Comm.

// The library's NCCL communicator (gnncg_comm_t).  Rank 0 calls unique_id() and the caller
// distributes the 128 bytes (MPI, a file, a TCP store ...); or wrap an existing ncclComm_t.
class Comm {
 public:
  static std::vector<char> unique_id() {
    std::vector<char> id(128);
    check(gnncg_comm_unique_id(id.data()), "gnncg_comm_unique_id");
    return id;
  }
  Comm(int nranks, int rank, const std::vector<char>& id) {
    if (id.size() != 128) throw std::invalid_argument("Comm: the unique id is 128 bytes");
    check(gnncg_comm_init(&c_, nranks, rank, id.data()), "gnncg_comm_init");
  }
  explicit Comm(void* nccl_comm) { check(gnncg_comm_init_nccl(&c_, nccl_comm), "gnncg_comm_init_nccl"); }
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  ~Comm() { gnncg_comm_destroy(c_); }
  int size() const { return gnncg_comm_size(c_); }
  int rank() const { return gnncg_comm_rank(c_); }
  gnncg_comm_t* get() const { return c_; }

 private:
  gnncg_comm_t* c_ = nullptr;
};

// Rank `rank`'s share of a P-way destination-row partition of a gnncg::Graph: rows
// [row_begin, row_end) = gnncg_partition_rows_weighted over the csr_dst offsets (cost-balanced), and
// the rank's in-edges split by the owner of their source (see gnncg_part_t).
class PartitionedGraph {
 public:
  // row_weight: the cost-balanced partitioner's per-row weight in edge units
  // (gnncg_partition_rows_weighted; 0 = edge-balanced blocks)
  PartitionedGraph(const Graph& g, int nparts, int rank, std::int32_t chunk = 2048, cudaStream_t stream = nullptr,
                   std::uint64_t row_weight = 64)
      : P_(nparts), rank_(rank), s_(stream) {
    check(gnncg_device_check(), "gnncg_device_check");
    if (nparts < 1 || rank < 0 || rank >= nparts) throw std::invalid_argument("PartitionedGraph: bad rank / nparts");
    const AdjIndex& in = g.csr_dst();
    const std::int64_t V = (std::int64_t)g.num_vertices();
    bounds_.resize(P_ + 1);
    check(gnncg_partition_rows_weighted(V, in.offsets.data(), P_, row_weight, bounds_.data()),
          "gnncg_partition_rows_weighted");
    for (int q = 0; q < P_; ++q) maxrows_ = std::max<std::int64_t>(maxrows_, bounds_[q + 1] - bounds_[q]);
    r0_ = (std::int64_t)bounds_[rank];
    n_ = (std::int64_t)bounds_[rank + 1] - r0_;
    const std::int64_t base = rank * maxrows_, Vp = P_ * maxrows_;
    // the rank's in-edges (csr_dst rows r0.., edge-id order), split by source owner
    std::vector<std::uint32_t> kl, ol, kr, orr;
    for (std::int64_t v = 0; v < n_; ++v)
      for (auto i = in.offsets[r0_ + v]; i < in.offsets[r0_ + v + 1]; ++i) {
        const std::uint64_t u = in.entries[i].vertex;
        const int q = (int)(std::upper_bound(bounds_.begin() + 1, bounds_.end(), u) - (bounds_.begin() + 1));
        const std::uint32_t pid = (std::uint32_t)(q * maxrows_ + (std::int64_t)(u - bounds_[q]));
        if (q == rank) {
          kl.push_back((std::uint32_t)v);
          ol.push_back(pid);
        } else {
          kr.push_back((std::uint32_t)v);
          orr.push_back(pid);
        }
      }
    DeviceBuffer ws;
    auto two = [&](DeviceIndex& csr, DeviceIndex& csc, std::vector<std::uint32_t>& dst, std::vector<std::uint32_t>& src,
                   std::int64_t csc_rows, std::int64_t shift) {
      DeviceBuffer dk = upload(dst.data(), dst.size(), s_);
      for (auto& x : src) x -= (std::uint32_t)shift;  // csc_local rows are rebased to the block
      DeviceBuffer sk = upload(src.data(), src.size(), s_);
      DeviceGraph::build_index(csc, csc_rows, n_, (std::int64_t)src.size(), sk.get<std::uint32_t>(),
                               dk.get<std::uint32_t>(), ws, chunk, s_);
      for (auto& x : src) x += (std::uint32_t)shift;
      DeviceBuffer sk2 = upload(src.data(), src.size(), s_);
      DeviceGraph::build_index(csr, n_, Vp, (std::int64_t)dst.size(), dk.get<std::uint32_t>(),
                               sk2.get<std::uint32_t>(), ws, chunk, s_);
    };
    two(csr_l_, csc_l_, kl, ol, n_, base);
    two(csr_r_, csc_r_, kr, orr, Vp, 0);
    views_[0] = csr_l_.view(); views_[1] = csr_r_.view(); views_[2] = csc_l_.view(); views_[3] = csc_r_.view();
    part_ = gnncg_part_t{n_, maxrows_, P_, rank_, &views_[0], &csr_l_.sched, &views_[1], &csr_r_.sched,
                         &views_[2], &csc_l_.sched, &views_[3], &csc_r_.sched, bounds_.data()};
  }
  PartitionedGraph(const PartitionedGraph&) = delete;
  PartitionedGraph& operator=(const PartitionedGraph&) = delete;

  int nparts() const { return P_; }
  int rank() const { return rank_; }
  std::int64_t row_begin() const { return r0_; }
  std::int64_t num_local() const { return n_; }
  std::int64_t maxrows() const { return maxrows_; }
  const gnncg_part_t* part() const { return &part_; }
  cudaStream_t stream() const { return s_; }
  DeviceBuffer& workspace(size_t bytes) const {
    ws_.ensure(bytes);
    return ws_;
  }

 private:
  int P_, rank_;
  cudaStream_t s_;
  std::vector<std::uint64_t> bounds_;
  std::int64_t maxrows_ = 0, r0_ = 0, n_ = 0;
  DeviceIndex csr_l_, csr_r_, csc_l_, csc_r_;
  gnncg_index_t views_[4];
  gnncg_part_t part_{};
  mutable DeviceBuffer ws_;
};

// Forward state of a rank: the gathered source tables (padded layout) and its rows' stash.
struct DistStash {
  DeviceBuffer Ht_all, Al_all, Ar, m, d, out;
};

namespace detail {
inline void require_comm(const PartitionedGraph& pg, const Comm* comm) {
  if (!comm && pg.nparts() > 1) throw std::invalid_argument("gat_*_dist: nparts > 1 needs a Comm");
  if (comm && comm->size() != pg.nparts()) throw std::invalid_argument("gat_*_dist: Comm size != nparts");
}
}  // namespace detail

// GAT layer forward of one rank: H_local = the rank's rows of H; returns its rows of out.
inline Tensor<float> gat_forward_dist(const PartitionedGraph& pg, const Comm* comm, const Tensor<float>& H_local,
                                      const Tensor<float>& W, const Tensor<float>& a_l, const Tensor<float>& a_r,
                                      const GatParams& p, DistStash* stash) {
  detail::require_comm(pg, comm);
  const std::int64_t n = pg.num_local(), h = p.heads, f = p.f, hf = h * f, Vp = pg.nparts() * pg.maxrows();
  const std::int64_t base = pg.rank() * pg.maxrows();
  detail::require_shape(H_local, n, H_local.cols, "gat_forward_dist H");
  detail::require_shape(W, H_local.cols, hf, "gat_forward_dist W");
  detail::require_shape(a_l, h, f, "gat_forward_dist a_l");
  detail::require_shape(a_r, h, f, "gat_forward_dist a_r");
  cudaStream_t s = pg.stream();
  DistStash local;
  DistStash& st = stash ? *stash : local;
  DeviceBuffer dH = upload(H_local, s), dW = upload(W, s), dal = upload(a_l, s), dar = upload(a_r, s);
  st.Ht_all = DeviceBuffer(std::max<std::int64_t>(Vp, 1) * hf * 4);
  st.Al_all = DeviceBuffer(std::max<std::int64_t>(Vp, 1) * h * 4);
  const std::int64_t nn = std::max<std::int64_t>(n, 1);
  st.Ar = DeviceBuffer(nn * h * 4);
  st.m = DeviceBuffer(nn * h * 4);
  st.d = DeviceBuffer(nn * h * 4);
  st.out = DeviceBuffer(nn * hf * 4);
  if (n > 0) {  // K1 into this rank's block of the gather tables
    DeviceBuffer& gws = pg.workspace(gnncg_gemm_workspace(0, 0, n, hf, H_local.cols));
    check(gnncg_gat_transform(n, H_local.cols, h, f, dH.get<float>(), H_local.cols, dW.get<float>(),
                              st.Ht_all.get<float>() + base * hf, dal.get<float>(), dar.get<float>(),
                              st.Al_all.get<float>() + base * h, st.Ar.get<float>(), gws.get(), gws.bytes(), s),
          "gnncg_gat_transform");
  }
  DeviceBuffer& ws = pg.workspace(gnncg_gat_dist_workspace(pg.part(), h, f));
  check(gnncg_gat_fwd_dist(comm ? comm->get() : nullptr, pg.part(), h, f, p.slope, st.Ht_all.get<float>(),
                           st.Al_all.get<float>(), st.Ar.get<float>(), st.out.get<float>(), st.m.get<float>(),
                           st.d.get<float>(), ws.get(), ws.bytes(), s),
        "gnncg_gat_fwd_dist");
  return download(st.out, n, hf, s);
}

// GAT layer backward of one rank (fused fast mode): dW / da_l / da_r are summed over the ranks
// (all-reduce); dH is the rank's rows.
inline GatGrads gat_backward_dist(const PartitionedGraph& pg, const Comm* comm, const Tensor<float>& H_local,
                                  const Tensor<float>& W, const Tensor<float>& a_l, const Tensor<float>& a_r,
                                  const DistStash& st, const Tensor<float>& dOut_local, const GatParams& p,
                                  bool need_dH) {
  detail::require_comm(pg, comm);
  const std::int64_t n = pg.num_local(), h = p.heads, f = p.f, hf = h * f, Fin = H_local.cols;
  const std::int64_t Vp = pg.nparts() * pg.maxrows(), base = pg.rank() * pg.maxrows(), nn = std::max<std::int64_t>(n, 1);
  detail::require_shape(dOut_local, n, hf, "gat_backward_dist dOut");
  detail::require_shape(W, Fin, hf, "gat_backward_dist W");
  cudaStream_t s = pg.stream();
  DeviceBuffer dH_in = upload(H_local, s), dW_in = upload(W, s), dal = upload(a_l, s), dar = upload(a_r, s);
  DeviceBuffer g_out = upload(dOut_local, s);
  DeviceBuffer dHt(nn * hf * 4), dAl(nn * h * 4), dAr(nn * h * 4);
  DeviceBuffer sendH(std::max<std::int64_t>(Vp, 1) * hf * 4), sendAl(std::max<std::int64_t>(Vp, 1) * h * 4);
  DeviceBuffer packed((Fin * hf + 2 * hf) * 4);
  float* dW = packed.get<float>();
  float* da_l = dW + Fin * hf;
  float* da_r = da_l + hf;
  {
    DeviceBuffer& ws = pg.workspace(gnncg_gat_dist_workspace(pg.part(), h, f));
    check(gnncg_gat_bwd_dist(comm ? comm->get() : nullptr, pg.part(), h, f, p.slope, st.Ht_all.get<float>(),
                             st.Al_all.get<float>(), st.Ar.get<float>(), st.m.get<float>(), st.d.get<float>(),
                             st.out.get<float>(), g_out.get<float>(), dal.get<float>(), dar.get<float>(),
                             dHt.get<float>(), dAl.get<float>(), dAr.get<float>(), sendH.get<float>(),
                             sendAl.get<float>(), ws.get(), ws.bytes(), s),
          "gnncg_gat_bwd_dist");
  }
  {
    DeviceBuffer& ws = pg.workspace(gnncg_gat_attn_grad_workspace(n, h, f));
    check(gnncg_gat_attn_grad(n, h, f, st.Ht_all.get<float>() + base * hf, dAl.get<float>(), dAr.get<float>(), da_l,
                              da_r, ws.get(), ws.bytes(), s),
          "gnncg_gat_attn_grad");
  }
  {
    DeviceBuffer& ws = pg.workspace(gnncg_gemm_workspace(1, 0, Fin, hf, n));
    check(gnncg_gemm(1, 0, Fin, hf, n, dH_in.get<float>(), Fin, dHt.get<float>(), hf, dW, hf, ws.get(), ws.bytes(), s),
          "gnncg_gemm");
  }
  if (comm) check(gnncg_comm_allreduce(comm->get(), dW, Fin * hf + 2 * hf, s), "gnncg_comm_allreduce");
  GatGrads out;
  const Tensor<float> all = download(packed, 1, Fin * hf + 2 * hf, s);
  out.dW = Tensor<float>(Fin, hf);
  out.da_l = Tensor<float>(h, f);
  out.da_r = Tensor<float>(h, f);
  std::copy(all.data.begin(), all.data.begin() + Fin * hf, out.dW.data.begin());
  std::copy(all.data.begin() + Fin * hf, all.data.begin() + Fin * hf + hf, out.da_l.data.begin());
  std::copy(all.data.begin() + Fin * hf + hf, all.data.end(), out.da_r.data.begin());
  if (need_dH) {
    DeviceBuffer dHb(nn * Fin * 4);
    DeviceBuffer& ws = pg.workspace(gnncg_gemm_workspace(0, 1, n, Fin, hf));
    check(gnncg_gemm(0, 1, n, Fin, hf, dHt.get<float>(), hf, dW_in.get<float>(), hf, dHb.get<float>(), Fin, ws.get(),
                     ws.bytes(), s),
          "gnncg_gemm");
    out.dH = download(dHb, n, Fin, s);
  }
  return out;
}

}  // namespace b200
}  // namespace gnncg
