// Microbenchmark (not product code): Zipf row gathers (1 KB fp32 rows of a 239 MB table, the
// Reddit-shaped K2 access stream) with neighbour ids prefetched a block ahead, so each warp
// keeps exactly U rows in flight; sweeps warps/SM x U to separate TLP from bytes in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench2 gather_bench2.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

template <int U>
__global__ void gather(const float4* __restrict__ table, const uint32_t* __restrict__ idx, int64_t nblk, float4* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float4 a0 = make_float4(0, 0, 0, 0), a1 = a0;
  int64_t b = warp;
  uint32_t id = b < nblk ? __ldg(idx + b * 32 + lane) : 0;
  for (; b < nblk; b += nwarps) {
    const uint32_t nid = b + nwarps < nblk ? __ldg(idx + (b + nwarps) * 32 + lane) : 0;  // next block's ids
#pragma unroll
    for (int j = 0; j < 32; j += U) {
      float4 x[U][2];
#pragma unroll
      for (int t = 0; t < U; ++t) {
        const uint32_t r = __shfl_sync(0xffffffffu, id, j + t);
        x[t][0] = __ldg(table + (int64_t)r * 64 + lane);
        x[t][1] = __ldg(table + (int64_t)r * 64 + 32 + lane);
      }
#pragma unroll
      for (int t = 0; t < U; ++t) {
        a0.x = fmaf(x[t][0].x, 0.5f, a0.x); a0.y = fmaf(x[t][0].y, 0.5f, a0.y);
        a0.z = fmaf(x[t][0].z, 0.5f, a0.z); a0.w = fmaf(x[t][0].w, 0.5f, a0.w);
        a1.x = fmaf(x[t][1].x, 0.5f, a1.x); a1.y = fmaf(x[t][1].y, 0.5f, a1.y);
        a1.z = fmaf(x[t][1].z, 0.5f, a1.z); a1.w = fmaf(x[t][1].w, 0.5f, a1.w);
      }
    }
    id = nid;
  }
  if (a0.x + a1.x == 123.456f) out[0] = a0;
}

template <int U>
void run(const float4* t, const uint32_t* idx, int64_t nblk, float4* out, int warps_per_sm) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 128;  // 4 warps per CTA
  const int grid = sms * warps_per_sm / 4;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather<U><<<grid, threads>>>(t, idx, nblk, out);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) gather<U><<<grid, threads>>>(t, idx, nblk, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, gather<U>, threads, 0);
  printf("U=%2d warps/SM=%2d (resident max %2d): %.3f ms  %.2f TB/s  rows-in-flight/SM=%d\n", U, warps_per_sm, nb * 4, ms,
         nblk * 32 * 1024.0 / ms / 1e9, U * warps_per_sm);
}

int main() {
  const int64_t V = 233000, E = 114000000 / 32 * 32;
  float4* table;
  uint32_t* idx;
  float4* out;
  cudaMalloc(&table, V * 1024);
  cudaMalloc(&idx, E * 4);
  cudaMalloc(&out, 64);
  cudaMemset(table, 0, V * 1024);
  std::vector<uint32_t> h(E);
  std::vector<double> cdf(V);
  double s = 0;
  for (int64_t i = 0; i < V; ++i) { s += 1.0 / (i + 1100.0); cdf[i] = s; }
  uint64_t st = 88172645463325252ull;
  for (int64_t e = 0; e < E; ++e) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    const double r = (st >> 11) * (1.0 / 9007199254740992.0) * s;
    int64_t lo = 0, hi = V - 1;
    while (lo < hi) { const int64_t m = (lo + hi) / 2; if (cdf[m] > r) hi = m; else lo = m + 1; }
    h[e] = (uint32_t)lo;
  }
  cudaMemcpy(idx, h.data(), E * 4, cudaMemcpyHostToDevice);
  const int64_t nblk = E / 32;
  for (int w : {16, 24, 32, 48, 64}) {
    run<2>(table, idx, nblk, out, w);
    run<4>(table, idx, nblk, out, w);
    run<8>(table, idx, nblk, out, w);
    if (w <= 32) run<16>(table, idx, nblk, out, w);
  }
  // L2 tiling probe: the same stream split into source tiles processed one after the other
  // (ids of tile t restricted to [t V/T, (t+1) V/T), each tile's rows ~ 239/T MB), vs one pass
  for (int T : {1, 2, 3, 4}) {
    std::vector<uint32_t> hs(h);
    // stable bucket by tile: a tile's edges are contiguous in the stream (2D-tiled order)
    std::vector<int64_t> cnt(T + 1, 0);
    for (int64_t e = 0; e < E; ++e) cnt[1 + (int64_t)h[e] * T / V]++;
    for (int t = 0; t < T; ++t) cnt[t + 1] += cnt[t];
    for (int64_t e = 0; e < E; ++e) hs[cnt[(int64_t)h[e] * T / V]++] = h[e];
    cudaMemcpy(idx, hs.data(), E * 4, cudaMemcpyHostToDevice);
    printf("tiles=%d: ", T);
    run<8>(table, idx, nblk, out, 16);
  }
  return 0;
}
