// Microbenchmark (not product code): how fast can B200 gather 1 KB rows of a
// 239 MB fp32 table by index?  Separates "our kernel is latency-bound" from
// "the L2/fabric path is the ceiling" for the GAT gather kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

template <int U>
__global__ void gather(const float4* __restrict__ table, const uint32_t* __restrict__ idx, int64_t n, float4* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t b = warp * U; b < n; b += nwarps * U) {
    float4 x[U][2];
#pragma unroll
    for (int t = 0; t < U; ++t) {
      const uint32_t r = (b + t < n) ? __ldg(idx + b + t) : 0;
      x[t][0] = __ldg(table + (int64_t)r * 64 + lane);
      x[t][1] = __ldg(table + (int64_t)r * 64 + 32 + lane);
    }
#pragma unroll
    for (int t = 0; t < U; ++t) {
      acc.x += x[t][0].x + x[t][1].x;
      acc.y += x[t][0].y + x[t][1].y;
      acc.z += x[t][0].z + x[t][1].z;
      acc.w += x[t][0].w + x[t][1].w;
    }
  }
  if (acc.x == 123.456f) out[0] = acc;
}

template <int U>
void run(const float4* t, const uint32_t* idx, int64_t n, float4* out, const char* name, int blocks_per_sm) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather<U><<<sms * blocks_per_sm, 256>>>(t, idx, n, out);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) gather<U><<<sms * blocks_per_sm, 256>>>(t, idx, n, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  printf("%-8s U=%2d blocks/SM=%d: %.3f ms  %.2f TB/s (rows)\n", name, U, blocks_per_sm, ms, n * 1024.0 / ms / 1e9);
}


// cp.async (LDGSTS) variant: rows land in a per-warp shared-memory ring without holding
// registers while in flight; NG groups of G rows per warp, consumed from shared memory.
template <int G, int NG>
__global__ void gather_async(const float4* __restrict__ table, const uint32_t* __restrict__ idx, int64_t n,
                             float4* out) {
  extern __shared__ float4 ring[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4* my = ring + (size_t)w * NG * G * 64;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  // this warp's groups: b = (warp + k*nwarps) * G, k = 0, 1, ...
  const int64_t ngroups = (n + G - 1) / G;
  auto issue = [&](int64_t k, int slot) {
    const int64_t gidx = warp + k * nwarps;
    if (gidx < ngroups) {
      const int64_t b = gidx * G;
#pragma unroll
      for (int t = 0; t < G; ++t) {
        const uint32_t r = (b + t < n) ? __ldg(idx + b + t) : 0;
        const float4* src = table + (int64_t)r * 64;
        float4* dst = my + (slot * G + t) * 64;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + q * 32 + lane);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src + q * 32 + lane));
        }
      }
    }
    asm volatile("cp.async.commit_group;");
  };
#pragma unroll
  for (int k = 0; k < NG - 1; ++k) issue(k, k);
  for (int64_t k = 0; warp + k * nwarps < ngroups; ++k) {
    asm volatile("cp.async.wait_group %0;" ::"n"(NG - 2));
    __syncwarp();
    const int slot = (int)(k % NG);
#pragma unroll
    for (int t = 0; t < G; ++t)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float4 x = my[(slot * G + t) * 64 + q * 32 + lane];
        acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
      }
    __syncwarp();
    issue(k + NG - 1, (int)((k + NG - 1) % NG));
  }
  asm volatile("cp.async.wait_all;");
  if (acc.x == 123.456f) out[0] = acc;
}

template <int G, int NG>
void run_async(const float4* t, const uint32_t* idx, int64_t n, float4* out, const char* name, int warps_per_block,
               int blocks_per_sm) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = (size_t)warps_per_block * NG * G * 1024;
  cudaFuncSetAttribute(gather_async<G, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather_async<G, NG><<<sms * blocks_per_sm, warps_per_block * 32, smem>>>(t, idx, n, out);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) gather_async<G, NG><<<sms * blocks_per_sm, warps_per_block * 32, smem>>>(t, idx, n, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  cudaError_t e = cudaGetLastError();
  printf("%-8s async G=%d NG=%d warps/SM=%d (%zu KB smem/CTA): %.3f ms  %.2f TB/s %s\n", name, G, NG,
         warps_per_block * blocks_per_sm, smem / 1024, ms, n * 1024.0 / ms / 1e9, e ? cudaGetErrorString(e) : "");
}

int main() {
  const int64_t V = 233000, E = 114000000;
  float4* table;
  uint32_t* idx;
  float4* out;
  cudaMalloc(&table, V * 1024);
  cudaMalloc(&idx, E * 4);
  cudaMalloc(&out, 64);
  cudaMemset(table, 0, V * 1024);
  std::vector<uint32_t> h(E);
  // Zipf-like (the bench graph's source distribution): P(i) ~ 1/(i+1100), sampled via the CDF
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
  for (int bps : {2, 4, 8}) {
    run<4>(table, idx, E, out, "zipf", bps);
    run<8>(table, idx, E, out, "zipf", bps);
    run<16>(table, idx, E, out, "zipf", bps);
  }
  run_async<4, 3>(table, idx, E, out, "zipf", 8, 2);   // 16 warps, 12 rows/warp
  run_async<4, 4>(table, idx, E, out, "zipf", 8, 2);   // 16 warps, 16 rows/warp (128 KB)
  run_async<2, 3>(table, idx, E, out, "zipf", 8, 4);   // 32 warps, 6 rows/warp
  run_async<2, 4>(table, idx, E, out, "zipf", 8, 4);   // 32 warps, 8 rows/warp (256 KB) -> 3 CTAs
  run_async<2, 3>(table, idx, E, out, "zipf", 16, 3);  // 48 warps, 6 rows/warp
  run_async<1, 4>(table, idx, E, out, "zipf", 16, 4);  // 64 warps, 4 rows/warp
  run_async<2, 2>(table, idx, E, out, "zipf", 16, 4);  // 64 warps, 4 rows/warp
  run_async<4, 3>(table, idx, E, out, "zipf", 4, 4);   // 16 warps in 4 CTAs
  for (int64_t e = 0; e < E; ++e) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; h[e] = (uint32_t)(st % V); }
  cudaMemcpy(idx, h.data(), E * 4, cudaMemcpyHostToDevice);
  for (int bps : {2, 4, 8}) {
    run<8>(table, idx, E, out, "uniform", bps);
    run<16>(table, idx, E, out, "uniform", bps);
  }
  // sequential (no gather): idx = e % V
  for (int64_t e = 0; e < E; ++e) h[e] = (uint32_t)(e % V);
  cudaMemcpy(idx, h.data(), E * 4, cudaMemcpyHostToDevice);
  run<8>(table, idx, E, out, "seq", 4);
  return 0;
}
