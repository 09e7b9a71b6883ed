// SPDX-License-Identifier: Apache-2.0
// Runtime plumbing of the C ABI: errors, device check, host-side schedule and
// partition construction (no device work here).
#include <atomic>
#include <cstdarg>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace gnncg_b200 {

static thread_local char g_err[1024] = "";
static std::atomic<unsigned long long> g_launches{0};
static std::atomic<unsigned long long*> g_cost{nullptr};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

unsigned long long* cost_slot(int kind) {
  unsigned long long* c = g_cost.load(std::memory_order_acquire);
  return c ? c + 2 * kind : nullptr;
}

__global__ void cost_add_kernel(unsigned long long* c, unsigned long long a, unsigned long long b) {
  c[0] += a;
  c[1] += b;
}

void cost_add(int kind, uint64_t a, uint64_t b, cudaStream_t s) {
  unsigned long long* c = cost_slot(kind);
  if (!c) return;
  cost_add_kernel<<<1, 1, 0, s>>>(c, a, b);
  note_launch();
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

int require_device() {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(GNNCG_ERR_NO_DEVICE, "no CUDA device: %s (gnncg_b200 has no CPU fallback)", cudaGetErrorString(e));
  }
  // Cache the capability per device ordinal.
  static thread_local int cached_dev = -2, cached_ok = 0;
  if (cached_dev != dev) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    cached_dev = dev;
    cached_ok = (major == 10 && minor == 0);
    if (!cached_ok)
      return fail(GNNCG_ERR_NO_DEVICE, "device %d is sm_%d%d; this library is built for sm_100a (B200) only", dev,
                  major, minor);
  }
  return cached_ok ? GNNCG_OK : fail(GNNCG_ERR_NO_DEVICE, "device %d is not sm_100", dev);
}

}  // namespace gnncg_b200

using namespace gnncg_b200;

extern "C" {

const char* gnncg_last_error(void) { return g_err; }

const char* gnncg_version(void) { return "gnncg_b200 0.1.0 (sm_100a)"; }

int gnncg_device_check(void) { return require_device(); }

uint64_t gnncg_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int gnncg_cost_counters(uint64_t* counters) {
  g_cost.store(reinterpret_cast<unsigned long long*>(counters), std::memory_order_release);
  return GNNCG_OK;
}

// Partitioner: bound[p] = lower_bound(off, ceil(p*E/P)).  Bit-exact with
// oracle/oracle.cpp:orc_partition_rows.
int gnncg_partition_rows(int64_t num_rows, const uint64_t* off, int32_t parts, uint64_t* bound) {
  GNNCG_REQUIRE(off && bound, GNNCG_ERR_ARG, "partition_rows: null pointer");
  GNNCG_REQUIRE(parts >= 1, GNNCG_ERR_ARG, "partition_rows: parts must be >= 1");
  const uint64_t V = (uint64_t)num_rows, E = off[V];
  bound[0] = 0;
  for (int p = 1; p < parts; ++p) {
    const uint64_t target = ((uint64_t)p * E + (uint64_t)parts - 1) / (uint64_t)parts;
    uint64_t lo = 0, hi = V + 1;  // lower_bound over off[0..V]
    while (lo < hi) {
      const uint64_t mid = (lo + hi) / 2;
      if (off[mid] < target) lo = mid + 1; else hi = mid;
    }
    bound[p] = lo > V ? V : lo;
    if (bound[p] < bound[p - 1]) bound[p] = bound[p - 1];
  }
  bound[parts] = V;
  return GNNCG_OK;
}

// Work items of the unified thread mapping (one warp per item):
//   * split rows (deg > chunk) first, each as ceil(deg/chunk) consecutive items
//     (hub rows start first: longest-processing-time order);
//   * then every other row (including empty rows, which must still write their
//     identity outputs) in descending log2-degree buckets, row order within a
//     bucket (deterministic counting sort, O(V)).
int gnncg_sched_build_host(int64_t num_rows, const uint64_t* off, int32_t chunk, int64_t* num_items,
                           int64_t* num_split_items, int64_t* num_split_rows, uint32_t* items,
                           uint32_t* split_rows, uint32_t* split_first) {
  GNNCG_REQUIRE(off && num_items && num_split_items && num_split_rows, GNNCG_ERR_ARG, "sched: null pointer");
  GNNCG_REQUIRE(chunk >= 32, GNNCG_ERR_ARG, "sched: chunk must be >= 32");
  GNNCG_REQUIRE(num_rows < (int64_t)0xFFFFFFFF, GNNCG_ERR_RANGE, "sched: too many rows for u32 ids");
  const int64_t V = num_rows;
  int64_t n_split_items = 0, n_split_rows = 0, n_items = 0;
  for (int64_t r = 0; r < V; ++r) {
    const uint64_t deg = off[r + 1] - off[r];
    if (deg > (uint64_t)chunk) {
      const int64_t n = (int64_t)((deg + chunk - 1) / chunk);
      n_split_items += n;
      n_split_rows += 1;
      n_items += n;
    } else {
      n_items += 1;
    }
  }
  *num_items = n_items;
  *num_split_items = n_split_items;
  *num_split_rows = n_split_rows;
  if (!items) return GNNCG_OK;
  GNNCG_REQUIRE(split_first && (n_split_rows == 0 || split_rows), GNNCG_ERR_ARG, "sched: null output array");
  int64_t it = 0, sr = 0;
  for (int64_t r = 0; r < V; ++r) {
    const uint64_t deg = off[r + 1] - off[r];
    if (deg > (uint64_t)chunk) {
      const int64_t n = (int64_t)((deg + chunk - 1) / chunk);
      split_rows[sr] = (uint32_t)r;
      split_first[sr] = (uint32_t)it;
      ++sr;
      for (int64_t c = 0; c < n; ++c) {
        items[2 * it] = (uint32_t)r;
        items[2 * it + 1] = (uint32_t)c;
        ++it;
      }
    }
  }
  split_first[sr] = (uint32_t)it;
  // Remaining rows: bucket by floor(log2(deg+1)), largest bucket first.
  int64_t count[40] = {0};
  auto bucket = [](uint64_t deg) {
    int b = 0;
    uint64_t x = deg + 1;
    while (x > 1) { x >>= 1; ++b; }
    return 39 - b;  // descending degree
  };
  for (int64_t r = 0; r < V; ++r) {
    const uint64_t deg = off[r + 1] - off[r];
    if (deg <= (uint64_t)chunk) count[bucket(deg)]++;
  }
  int64_t start[40];
  int64_t acc = it;
  for (int b = 0; b < 40; ++b) { start[b] = acc; acc += count[b]; }
  for (int64_t r = 0; r < V; ++r) {
    const uint64_t deg = off[r + 1] - off[r];
    if (deg <= (uint64_t)chunk) {
      const int64_t p = start[bucket(deg)]++;
      items[2 * p] = (uint32_t)r;
      items[2 * p + 1] = 0u;
    }
  }
  return GNNCG_OK;
}

}  // extern "C"
