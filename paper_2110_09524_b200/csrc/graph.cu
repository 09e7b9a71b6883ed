// SPDX-License-Identifier: Apache-2.0
//
// Graph store on the device (K9): CSR/CSC construction bit-identical to the
// reference's build_index (proj/src/graph.cpp:14-28), a deterministic
// Chung-Lu power-law edge generator, and a max-degree reduction
// (degree_stats, graph.cpp:47-57).
//
// build_index is a counting sort stable in edge id.  On the device the same
// order is obtained by radix-sorting the unique 64-bit keys (key_vertex << 32 |
// edge_id): with unique keys any correct sort is the stable one, so the result
// is bit-identical to the reference for every input.  Offsets are then read off
// the sorted keys by a boundary scan (empty rows included).
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace gnncg_b200 {
namespace {

__global__ void make_keys_kernel(int64_t E, int64_t V, int64_t n_other, const uint32_t* __restrict__ key,
                                 const uint32_t* __restrict__ other, uint64_t* __restrict__ keys,
                                 int* __restrict__ bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = key[e];
    if (k >= (uint64_t)V || other[e] >= (uint64_t)n_other) atomicOr(bad, 1);  // graph.cpp:37-39
    keys[e] = ((uint64_t)k << 32) | (uint64_t)(uint32_t)e;
  }
}

// off[r] = first sorted position whose key vertex >= r.
__global__ void offsets_kernel(int64_t E, int64_t V, const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ other,
                               uint64_t* __restrict__ off, uint32_t* __restrict__ nbr, uint32_t* __restrict__ eid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= E; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i < E ? (int64_t)(skeys[i] >> 32) : V;  // sentinel: rows after the last key end at E
    const int64_t vp = i > 0 ? (int64_t)(skeys[i - 1] >> 32) : -1;
    for (int64_t r = vp + 1; r <= v && r <= V; ++r) off[r] = (uint64_t)i;
    if (i < E) {
      const uint32_t e = (uint32_t)(skeys[i] & 0xFFFFFFFFu);
      eid[i] = e;
      nbr[i] = other[e];
    }
  }
}

__global__ void max_degree_kernel(int64_t rows, const uint64_t* __restrict__ off, unsigned long long* __restrict__ out) {
  uint64_t best = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
    best = max(best, off[r + 1] - off[r]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = max(best, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)best, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)best);
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// smallest i with cdf[i] > r  (cdf inclusive, strictly increasing for positive weights)
__device__ __forceinline__ uint32_t sample_cdf(const uint64_t* __restrict__ cdf, int64_t V, uint64_t r) {
  int64_t lo = 0, hi = V - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(cdf + mid) > r) hi = mid; else lo = mid + 1;
  }
  return (uint32_t)lo;
}

__global__ void chung_lu_kernel(int64_t V, int64_t E, const uint64_t* __restrict__ cdf, uint64_t seed,
                                uint32_t* __restrict__ src, uint32_t* __restrict__ dst) {
  const uint64_t total = cdf[V - 1];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h0 = splitmix64(seed * 0xD1B54A32D192ED03ull + 2ull * (uint64_t)e);
    const uint64_t h1 = splitmix64(seed * 0xD1B54A32D192ED03ull + 2ull * (uint64_t)e + 1ull);
    dst[e] = sample_cdf(cdf, V, __umul64hi(h0, total));
    src[e] = sample_cdf(cdf, V, __umul64hi(h1, total));
  }
}

__device__ __forceinline__ void chung_lu_edge(int64_t V, const uint64_t* __restrict__ cdf, uint64_t total,
                                              uint64_t seed, int64_t e, uint32_t& s, uint32_t& d) {
  const uint64_t h0 = splitmix64(seed * 0xD1B54A32D192ED03ull + 2ull * (uint64_t)e);
  const uint64_t h1 = splitmix64(seed * 0xD1B54A32D192ED03ull + 2ull * (uint64_t)e + 1ull);
  d = sample_cdf(cdf, V, __umul64hi(h0, total));
  s = sample_cdf(cdf, V, __umul64hi(h1, total));
}

// In-degree histogram of the generated edge list (the destination draw only).
__global__ void chung_lu_degree_kernel(int64_t V, int64_t E, const uint64_t* __restrict__ cdf, uint64_t seed,
                                       uint32_t* __restrict__ deg) {
  const uint64_t total = cdf[V - 1];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h0 = splitmix64(seed * 0xD1B54A32D192ED03ull + 2ull * (uint64_t)e);
    atomicAdd(deg + sample_cdf(cdf, V, __umul64hi(h0, total)), 1u);
  }
}

// Edges of one destination row block, in edge-id order (a rank's in-edges): tiles of
// kGenTile edges; pass 0 counts the kept edges of each tile, pass 1 (after an exclusive
// scan of the counts) writes them at the tile's offset in warp-ballot order.
constexpr int kGenTile = 4096;

template <bool WRITE>
__global__ void __launch_bounds__(256) chung_lu_rows_kernel(int64_t V, int64_t E, const uint64_t* __restrict__ cdf,
                                                            uint64_t seed, uint32_t r0, uint32_t r1,
                                                            uint64_t* __restrict__ tile_off, uint32_t* __restrict__ src,
                                                            uint32_t* __restrict__ dst) {
  __shared__ uint32_t wcount[8];
  const uint64_t total = cdf[V - 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t t0 = (int64_t)blockIdx.x * kGenTile;
  uint64_t pos = WRITE ? tile_off[blockIdx.x] : 0;
  uint32_t kept = 0;
  for (int64_t c = 0; c < kGenTile; c += 256) {
    const int64_t e = t0 + c + threadIdx.x;
    uint32_t s = 0, d = 0;
    bool keep = false;
    if (e < E) {
      chung_lu_edge(V, cdf, total, seed, e, s, d);
      keep = d >= r0 && d < r1;
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) wcount[w] = __popc(m);
    __syncthreads();
    if (WRITE) {
      uint32_t before = 0;
      for (int i = 0; i < w; ++i) before += wcount[i];
      if (keep) {
        const uint64_t at = pos + before + __popc(m & ((1u << lane) - 1u));
        src[at] = s;
        dst[at] = d;
      }
    }
    uint32_t all = 0;
    for (int i = 0; i < 8; ++i) all += wcount[i];
    pos += all;
    kept += all;
    __syncthreads();
  }
  if (!WRITE && threadIdx.x == 0) tile_off[blockIdx.x] = kept;
}

__global__ void exclusive_scan_serial_kernel(int64_t n, uint64_t* __restrict__ v) {
  // one thread block: n is E / 4096 (244K at 1B edges)
  __shared__ uint64_t part[1024];
  const int64_t per = ceil_div(n, (int64_t)blockDim.x);
  const int64_t b = threadIdx.x * per, e = min(n, b + per);
  uint64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += v[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t run = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const uint64_t t = part[i];
      part[i] = run;
      run += t;
    }
  }
  __syncthreads();
  uint64_t run = part[threadIdx.x];
  for (int64_t i = b; i < e; ++i) {
    const uint64_t t = v[i];
    v[i] = run;
    run += t;
  }
}

int grid_for(int64_t n, int threads = 256) {
  int64_t g = ceil_div(n > 0 ? n : 1, threads);
  return (int)(g > 148 * 64 ? 148 * 64 : g);
}

size_t sort_temp_bytes(int64_t E) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int)E, 0, 64);
  return bytes;
}

int bits_for(int64_t V) {
  int b = 1;
  while (b < 32 && ((int64_t)1 << b) <= V) ++b;
  return b;
}

}  // namespace
}  // namespace gnncg_b200

using namespace gnncg_b200;

extern "C" {

size_t gnncg_csr_build_workspace(int64_t V, int64_t E) {
  (void)V;
  return align_up(2 * (size_t)E * sizeof(uint64_t)) + align_up(sort_temp_bytes(E)) + 256;
}

int gnncg_csr_build(int64_t V, int64_t E, const uint32_t* key, const uint32_t* other, uint64_t* off, uint32_t* nbr,
                    uint32_t* eid, void* ws, size_t ws_bytes, void* stream) {
  return gnncg_csr_build_rect(V, V, E, key, other, off, nbr, eid, ws, ws_bytes, stream);
}

int gnncg_csr_build_rect(int64_t V, int64_t n_other, int64_t E, const uint32_t* key, const uint32_t* other,
                         uint64_t* off, uint32_t* nbr, uint32_t* eid, void* ws, size_t ws_bytes, void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(V >= 0 && E >= 0 && n_other >= 0, GNNCG_ERR_ARG, "csr_build: negative size");
  GNNCG_REQUIRE(n_other <= ((int64_t)1 << 32), GNNCG_ERR_RANGE, "csr_build: neighbour ids exceed u32");
  GNNCG_REQUIRE(E < ((int64_t)1 << 31), GNNCG_ERR_UNSUPPORTED, "csr_build: E >= 2^31 not supported by this build");
  GNNCG_REQUIRE(V < ((int64_t)1 << 32) - 1, GNNCG_ERR_RANGE, "csr_build: V exceeds u32 vertex ids");
  GNNCG_REQUIRE(off && (E == 0 || (key && other && nbr && eid)), GNNCG_ERR_ARG, "csr_build: null pointer");
  const size_t need = gnncg_csr_build_workspace(V, E);
  GNNCG_REQUIRE(ws_bytes >= need && ws, GNNCG_ERR_WORKSPACE, "csr_build: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = as_stream(stream);
  char* p = static_cast<char*>(ws);
  uint64_t* keys_in = reinterpret_cast<uint64_t*>(p);
  uint64_t* keys_out = keys_in + E;
  p += align_up(2 * (size_t)E * sizeof(uint64_t));
  void* temp = p;
  size_t temp_bytes = sort_temp_bytes(E);
  p += align_up(temp_bytes);
  int* bad = reinterpret_cast<int*>(p);
  GNNCG_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), s));
  if (E > 0) {
    make_keys_kernel<<<grid_for(E), 256, 0, s>>>(E, V, n_other, key, other, keys_in, bad);
    GNNCG_LAUNCH_CHECK();
    GNNCG_CUDA_TRY(cub::DeviceRadixSort::SortKeys(temp, temp_bytes, keys_in, keys_out, (int)E, 0, 32 + bits_for(V), s));
  }
  offsets_kernel<<<grid_for(E + 1), 256, 0, s>>>(E, V, keys_out, other, off, nbr, eid);
  GNNCG_LAUNCH_CHECK();
  int hbad = 0;
  GNNCG_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  GNNCG_CUDA_TRY(cudaStreamSynchronize(s));
  GNNCG_REQUIRE(!hbad, GNNCG_ERR_RANGE, "edge endpoint out of range");  // GraphError, graph.cpp:37-39
  return GNNCG_OK;
}

int gnncg_max_degree(const gnncg_index_t* idx, uint64_t* out_host, void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(idx && out_host, GNNCG_ERR_ARG, "max_degree: null pointer");
  cudaStream_t s = as_stream(stream);
  unsigned long long* d = nullptr;
  GNNCG_CUDA_TRY(cudaMallocAsync(&d, sizeof(unsigned long long), s));  // not a hot call
  GNNCG_CUDA_TRY(cudaMemsetAsync(d, 0, sizeof(unsigned long long), s));
  if (idx->num_rows > 0) {
    max_degree_kernel<<<grid_for(idx->num_rows), 256, 0, s>>>(idx->num_rows, idx->off, d);
    GNNCG_LAUNCH_CHECK();
  }
  unsigned long long h = 0;
  GNNCG_CUDA_TRY(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
  GNNCG_CUDA_TRY(cudaFreeAsync(d, s));
  GNNCG_CUDA_TRY(cudaStreamSynchronize(s));
  *out_host = (uint64_t)h;
  return GNNCG_OK;
}

int gnncg_gen_chung_lu_degrees(int64_t V, int64_t E, const uint64_t* cdf, uint64_t seed, uint32_t* in_deg,
                               void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(V > 0 && E >= 0 && cdf && in_deg, GNNCG_ERR_ARG, "gen_chung_lu_degrees: bad argument");
  cudaStream_t s = as_stream(stream);
  GNNCG_CUDA_TRY(cudaMemsetAsync(in_deg, 0, sizeof(uint32_t) * (size_t)V, s));
  if (E == 0) return GNNCG_OK;
  chung_lu_degree_kernel<<<grid_for(E), 256, 0, s>>>(V, E, cdf, seed, in_deg);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

size_t gnncg_gen_chung_lu_rows_workspace(int64_t E) {
  return align_up((size_t)ceil_div(E > 0 ? E : 1, kGenTile) * sizeof(uint64_t));
}

int gnncg_gen_chung_lu_rows(int64_t V, int64_t E, const uint64_t* cdf, uint64_t seed, int64_t row_begin,
                            int64_t row_end, uint32_t* src, uint32_t* dst, void* workspace, size_t workspace_bytes,
                            void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(V > 0 && E >= 0 && cdf && 0 <= row_begin && row_begin <= row_end && row_end <= V, GNNCG_ERR_ARG,
                "gen_chung_lu_rows: bad argument");
  if (E == 0 || row_begin == row_end) return GNNCG_OK;
  GNNCG_REQUIRE(src && dst, GNNCG_ERR_ARG, "gen_chung_lu_rows: null output");
  const size_t need = gnncg_gen_chung_lu_rows_workspace(E);
  GNNCG_REQUIRE(workspace && workspace_bytes >= need, GNNCG_ERR_WORKSPACE, "gen_chung_lu_rows: workspace %zu < %zu",
                workspace_bytes, need);
  cudaStream_t s = as_stream(stream);
  const int64_t tiles = ceil_div(E, kGenTile);
  GNNCG_REQUIRE(tiles < (int64_t)INT32_MAX, GNNCG_ERR_RANGE, "gen_chung_lu_rows: too many edges");
  uint64_t* tile_off = static_cast<uint64_t*>(workspace);
  chung_lu_rows_kernel<false><<<(unsigned)tiles, 256, 0, s>>>(V, E, cdf, seed, (uint32_t)row_begin, (uint32_t)row_end,
                                                              tile_off, nullptr, nullptr);
  GNNCG_LAUNCH_CHECK();
  exclusive_scan_serial_kernel<<<1, 1024, 0, s>>>(tiles, tile_off);
  GNNCG_LAUNCH_CHECK();
  chung_lu_rows_kernel<true><<<(unsigned)tiles, 256, 0, s>>>(V, E, cdf, seed, (uint32_t)row_begin, (uint32_t)row_end,
                                                             tile_off, src, dst);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

int gnncg_gen_chung_lu(int64_t V, int64_t E, const uint64_t* cdf, uint64_t seed, uint32_t* src, uint32_t* dst,
                       void* stream) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(V > 0 && E >= 0 && cdf && (E == 0 || (src && dst)), GNNCG_ERR_ARG, "gen_chung_lu: bad argument");
  if (E == 0) return GNNCG_OK;
  chung_lu_kernel<<<grid_for(E), 256, 0, as_stream(stream)>>>(V, E, cdf, seed, src, dst);
  GNNCG_LAUNCH_CHECK();
  return GNNCG_OK;
}

}  // extern "C"
