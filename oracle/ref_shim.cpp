// SPDX-License-Identifier: Apache-2.0
//
// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the reference's OWN graph and tensor code.  It is
// compiled together with /root/reference/proj/src/graph.cpp and tensor.cpp (left
// where they lie; see oracle/Makefile) into oracle/_ref/libgnncg_ref.so so that
// tests can pin the restated oracle and the device CSR builder to the reference's
// actual outputs:
//   * Graph::Graph / build_index     proj/src/graph.cpp:14-45   (bit-exact CSR/CSC)
//   * degree_stats                   proj/src/graph.cpp:47-57
//   * generate_synthetic(descriptor) proj/src/graph.cpp:157-249
//   * init_seeded<T>                 proj/include/gnncg/tensor.hpp:44-63
//   * matmul / matmul_nt / matmul_tn proj/src/tensor.cpp:8-60
//   * max_rel_err                    proj/include/gnncg/tensor.hpp:153-166
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "gnncg/graph.hpp"
#include "gnncg/tensor.hpp"

using gnncg::Graph;

namespace {
void set_err(char* err, int n, const char* msg) {
  if (err && n > 0) {
    std::strncpy(err, msg, (size_t)n - 1);
    err[n - 1] = 0;
  }
}
}  // namespace

extern "C" {

void* ref_graph_new(std::uint64_t V, std::uint64_t E, const std::uint32_t* src, const std::uint32_t* dst, char* err,
                    int errlen) {
  try {
    std::vector<std::pair<gnncg::VertexId, gnncg::VertexId>> edges(E);
    for (std::uint64_t e = 0; e < E; ++e) edges[e] = {src[e], dst[e]};
    return new Graph(V, std::move(edges));
  } catch (const std::exception& ex) {
    set_err(err, errlen, ex.what());
    return nullptr;
  }
}

void* ref_graph_synthetic(const char* descriptor, std::uint64_t seed, char* err, int errlen) {
  try {
    return new Graph(gnncg::generate_synthetic(std::string(descriptor), seed));
  } catch (const std::exception& ex) {
    set_err(err, errlen, ex.what());
    return nullptr;
  }
}

void* ref_graph_load_edge_list(const char* path, int undirected, char* err, int errlen) {
  try {
    return new Graph(gnncg::load_edge_list(std::string(path), undirected != 0));
  } catch (const std::exception& ex) {
    set_err(err, errlen, ex.what());
    return nullptr;
  }
}

void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }

void ref_graph_dims(const void* gp, std::uint64_t* V, std::uint64_t* E) {
  const Graph* g = static_cast<const Graph*>(gp);
  *V = g->num_vertices();
  *E = g->num_edges();
}

// which = 0: csr_dst (in-edges by destination), 1: csc_src (out-edges by source)
void ref_graph_index(const void* gp, int which, std::uint64_t* off, std::uint32_t* nbr, std::uint32_t* eid) {
  const Graph* g = static_cast<const Graph*>(gp);
  const gnncg::AdjIndex& idx = which == 0 ? g->csr_dst() : g->csc_src();
  for (std::size_t i = 0; i < idx.offsets.size(); ++i) off[i] = idx.offsets[i];
  for (std::size_t i = 0; i < idx.entries.size(); ++i) {
    nbr[i] = idx.entries[i].vertex;
    eid[i] = idx.entries[i].edge;
  }
}

void ref_graph_edges(const void* gp, std::uint32_t* src, std::uint32_t* dst) {
  const Graph* g = static_cast<const Graph*>(gp);
  for (std::uint64_t e = 0; e < g->num_edges(); ++e) {
    src[e] = g->edge_src(static_cast<gnncg::EdgeId>(e));
    dst[e] = g->edge_dst(static_cast<gnncg::EdgeId>(e));
  }
}

void ref_degree_stats(const void* gp, std::uint64_t* max_in, double* mean_in, std::uint64_t* max_out) {
  const gnncg::DegreeStats s = gnncg::degree_stats(*static_cast<const Graph*>(gp));
  *max_in = s.max_in_degree;
  *mean_in = s.mean_in_degree;
  *max_out = s.max_out_degree;
}

void ref_init_seeded_f64(std::uint64_t rows, std::uint64_t cols, std::uint64_t seed, int dist, double* out) {
  auto t = gnncg::init_seeded<double>(rows, cols, seed, static_cast<gnncg::InitDist>(dist));
  std::memcpy(out, t.data.data(), t.data.size() * sizeof(double));
}

void ref_init_seeded_f32(std::uint64_t rows, std::uint64_t cols, std::uint64_t seed, int dist, float* out) {
  auto t = gnncg::init_seeded<float>(rows, cols, seed, static_cast<gnncg::InitDist>(dist));
  std::memcpy(out, t.data.data(), t.data.size() * sizeof(float));
}

}  // extern "C"

template <typename T>
static gnncg::Tensor<T> wrap(std::uint64_t r, std::uint64_t c, const T* p) {
  gnncg::Tensor<T> t(r, c);
  std::memcpy(t.data.data(), p, r * c * sizeof(T));
  return t;
}

extern "C" {

// op: 0 = matmul (A[M,K] B[K,N]), 1 = matmul_nt (A[M,K] B[N,K]^T), 2 = matmul_tn (A[K,M]^T B[K,N])
int ref_matmul_f32(int op, std::uint64_t ar, std::uint64_t ac, const float* A, std::uint64_t br, std::uint64_t bc,
                   const float* B, float* C) {
  try {
    auto a = wrap(ar, ac, A);
    auto b = wrap(br, bc, B);
    gnncg::Tensor<float> c = op == 0 ? gnncg::matmul(a, b) : op == 1 ? gnncg::matmul_nt(a, b) : gnncg::matmul_tn(a, b);
    std::memcpy(C, c.data.data(), c.data.size() * sizeof(float));
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

int ref_matmul_f64(int op, std::uint64_t ar, std::uint64_t ac, const double* A, std::uint64_t br, std::uint64_t bc,
                   const double* B, double* C) {
  try {
    auto a = wrap(ar, ac, A);
    auto b = wrap(br, bc, B);
    gnncg::Tensor<double> c =
        op == 0 ? gnncg::matmul(a, b) : op == 1 ? gnncg::matmul_nt(a, b) : gnncg::matmul_tn(a, b);
    std::memcpy(C, c.data.data(), c.data.size() * sizeof(double));
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

double ref_max_rel_err_f64(std::uint64_t n, const double* a, const double* b) {
  return gnncg::max_rel_err(wrap<double>(1, n, a), wrap<double>(1, n, b));
}

}  // extern "C"
