// SPDX-License-Identifier: Apache-2.0
// Runtime plumbing of the C ABI: errors, device check, host-side schedule and
// partition construction (no device work here).
#include <algorithm>
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

static std::atomic<size_t> g_l2_persist{0};
size_t l2_persist_bytes() { return g_l2_persist.load(std::memory_order_relaxed); }

// argmax_b off[b+n] - off[b] (lowest b on ties), cached for the last few (off, rows, n): the
// scan is O(rows) on the host and a schedule is reused for every layer and step.
int64_t hot_window_begin(const uint64_t* off, int64_t rows, int64_t n) {
  if (!off || rows <= 0 || n <= 0 || n >= rows) return 0;
  struct Hit { const uint64_t* off; int64_t rows, n, b; };
  static thread_local Hit cache[4] = {};
  static thread_local int next = 0;
  for (const Hit& c : cache)
    if (c.off == off && c.rows == rows && c.n == n) return c.b;
  int64_t best = 0;
  uint64_t bv = off[n] - off[0];
  for (int64_t b = 1; b + n <= rows; ++b) {
    const uint64_t v = off[b + n] - off[b];
    if (v > bv) { bv = v; best = b; }
  }
  cache[next] = Hit{off, rows, n, best};
  next = (next + 1) % 4;
  return best;
}

// The window for a gather of `table` (rows of row_bytes) under schedule `sched`, or {null, 0}.
L2Window l2_window(const gnncg_sched_t* sched, const void* table, size_t row_bytes) {
  const size_t pb = l2_persist_bytes();
  if (pb == 0 || !sched || !sched->gather_off || sched->gather_rows <= 0 || !table || row_bytes == 0) return {};
  const int64_t n = std::min<int64_t>((int64_t)(pb / row_bytes), sched->gather_rows);
  if (n <= 0) return {};
  const int64_t b = hot_window_begin(sched->gather_off, sched->gather_rows, n);
  // only where the window concentrates the reads: at least twice its share of the rows.  A
  // shuffled labelling has no such range, and persisting an arbitrary slice of it was measured
  // slower than no window (C2: 39.6 vs 37.4 ms; degree-ordered ids: 35.0 ms with the window).
  const uint64_t* off = sched->gather_off;
  const double reads = (double)(off[b + n] - off[b]), total = (double)off[sched->gather_rows];
  if (total <= 0.0 || reads < 2.0 * total * (double)n / (double)sched->gather_rows) return {};
  return {static_cast<const char*>(table) + (size_t)b * row_bytes, (size_t)n * row_bytes};
}

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

int gnncg_l2_persist(size_t bytes, size_t* granted) {
  GNNCG_DEVICE_GUARD();
  int dev = 0, mx = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev);
  const size_t want = std::min<size_t>(bytes, (size_t)std::max(mx, 0));
  cudaError_t e = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
  if (e == cudaSuccess && want == 0) e = cudaCtxResetPersistingL2Cache();
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(GNNCG_ERR_CUDA, "l2_persist: %s", cudaGetErrorString(e));
  }
  g_l2_persist.store(want, std::memory_order_relaxed);
  if (granted) *granted = want;
  return GNNCG_OK;
}

int gnncg_hot_window_host(int64_t num_rows, const uint64_t* off, int64_t n, int64_t* begin) {
  GNNCG_REQUIRE(off && begin, GNNCG_ERR_ARG, "hot_window: null pointer");
  GNNCG_REQUIRE(num_rows >= 0 && n >= 0, GNNCG_ERR_ARG, "hot_window: negative size");
  *begin = hot_window_begin(off, num_rows, std::min(n, num_rows));
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

int gnncg_partition_rows_weighted(int64_t num_rows, const uint64_t* off, int32_t parts, uint64_t row_weight,
                                  uint64_t* bound) {
  GNNCG_REQUIRE(off && bound, GNNCG_ERR_ARG, "partition_rows_weighted: null pointer");
  GNNCG_REQUIRE(parts >= 1, GNNCG_ERR_ARG, "partition_rows_weighted: parts must be >= 1");
  const uint64_t V = (uint64_t)num_rows;
  const auto cost = [&](uint64_t v) { return off[v] + row_weight * v; };
  const uint64_t total = cost(V);
  bound[0] = 0;
  for (int p = 1; p < parts; ++p) {
    const uint64_t target = (uint64_t)(((unsigned __int128)p * total + (uint64_t)parts - 1) / (uint64_t)parts);
    uint64_t lo = 0, hi = V + 1;  // lower_bound over cost[0..V] (non-decreasing)
    while (lo < hi) {
      const uint64_t mid = (lo + hi) / 2;
      if (cost(mid) < target) lo = mid + 1; else hi = mid;
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
