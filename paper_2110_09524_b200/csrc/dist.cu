// SPDX-License-Identifier: Apache-2.0
//
// Multi-GPU GAT region of one rank (include/gnncg_b200.h "multi-GPU"; SURVEY §8(b), §8(e);
// north_star: destination-row partitioning, all-gather of the transformed features per layer).
//
// The reference's executor is single-process; this file adds what a rank
// needs on top of the single-GPU kernels:
//   * a communicator handle over NCCL, resolved with dlopen at run time (no link-time
//     dependency: a process that already loaded NCCL -- torch -- shares that copy);
//   * gnncg_gat_fwd_dist: the all-gather of Ht || A_l on the communicator's stream overlapped
//     with K2 over the rank's local-source edges, then K2 over the remote-source edges and an
//     online-softmax merge of the two partials;
//   * gnncg_gat_bwd_dist: K4f over the remote-source edges first, their reduce-scatter
//     overlapped with K4f over the local-source edges, then one combine pass.
// Why collectives and not peer loads inside K2: every source row is gathered E/V times per
// layer (489 at C2), so moving it once per layer over NVLink and then gathering from local
// HBM / L2 beats reading it from peer memory per edge.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "gat_internal.h"

namespace gnncg_b200 {
namespace {

// ------------------------------------------------------------------ NCCL at run time
struct NcclApi {
  bool ok = false;
  char why[256] = {0};
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    if (const char* path = std::getenv("GNNCG_NCCL_LIB")) h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's copy (torch's)
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      std::snprintf(api.why, sizeof(api.why), "libnccl.so.2 not loadable: %s", dlerror());
      return;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) all = false;
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.CommCount, "ncclCommCount");
    sym(api.CommUserRank, "ncclCommUserRank");
    sym(api.AllGather, "ncclAllGather");
    sym(api.ReduceScatter, "ncclReduceScatter");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.Broadcast, "ncclBroadcast");
    sym(api.Reduce, "ncclReduce");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
    if (!all) {
      std::snprintf(api.why, sizeof(api.why), "libnccl.so.2 lacks a required symbol");
      return;
    }
    api.ok = true;
  });
  return api;
}

#define GNNCG_NCCL_TRY(expr)                                                                              \
  do {                                                                                                    \
    ncclResult_t r__ = (expr);                                                                            \
    if (r__ != ncclSuccess)                                                                               \
      return ::gnncg_b200::fail(GNNCG_ERR_NCCL, "%s:%d %s: %s", __FILE__, __LINE__, #expr,               \
                                nccl().GetErrorString ? nccl().GetErrorString(r__) : "nccl error");      \
  } while (0)

#define GNNCG_NCCL_API()                                                                      \
  do {                                                                                        \
    if (!nccl().ok) return ::gnncg_b200::fail(GNNCG_ERR_NCCL, "NCCL unavailable: %s", nccl().why); \
  } while (0)

// ------------------------------------------------------------------ kernels
// Merge of two online-softmax partials of the same rows (K2 over disjoint edge sets):
// (outA, mA, dA) into (out, m, d) in place.  One warp per row: the row's (m, d) pairs are
// read into lanes (h <= 32) before any lane writes them.
template <int VW>
__global__ void __launch_bounds__(256) gat_merge2_kernel(int64_t rows, int h, int f, const float* __restrict__ outA,
                                                         const float* __restrict__ mA, const float* __restrict__ dA,
                                                         float* __restrict__ out, float* __restrict__ m,
                                                         float* __restrict__ d) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int hf = h * f;
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    float wa = 0.f, wb = 1.f, M = 0.f, D = 0.f;
    if (lane < h) {
      const float ma = mA[r * h + lane], da = dA[r * h + lane];
      const float mb = m[r * h + lane], db = d[r * h + lane];
      if (da == 0.f) {  // empty part A (m = d = 0)
        M = mb; D = db;
      } else if (db == 0.f) {
        wa = 1.f; wb = 0.f; M = ma; D = da;
      } else {
        M = fmaxf(ma, mb);
        const float ea = da * __expf(ma - M), eb = db * __expf(mb - M);
        D = ea + eb;
        wa = ea / D; wb = eb / D;
      }
    }
    __syncwarp();
    for (int c0 = 0; c0 < hf; c0 += 32 * VW) {
      const int c = c0 + lane * VW;
      const int k = (c < hf ? c : 0) / f;  // VW divides f: one head per vector
      const float a = __shfl_sync(0xffffffffu, wa, k), b = __shfl_sync(0xffffffffu, wb, k);
      if (c < hf) {
        const int64_t at = r * hf + c;
#pragma unroll
        for (int j = 0; j < VW; ++j) out[at + j] = fmaf(a, outA[at + j], b * out[at + j]);
      }
    }
    if (lane < h) {
      m[r * h + lane] = M;
      d[r * h + lane] = D;
    }
  }
}

// dHt[r,:] += recvH[r,:] + dA_r[r,k] a_r[k,:] ;  dAl[r,:] += recvAl[r,:]   (r < rows)
__global__ void __launch_bounds__(256) gat_dist_combine_kernel(int64_t rows, int h, int f,
                                                               const float* __restrict__ recvH,
                                                               const float* __restrict__ recvAl,
                                                               const float* __restrict__ dAr,
                                                               const float* __restrict__ a_r, float* __restrict__ dHt,
                                                               float* __restrict__ dAl) {
  const int hf = h * f;
  const int64_t n1 = rows * hf, n2 = rows * h;
  if ((f & 3) == 0 && (hf >> 2) <= (int)blockDim.x) {
    // threads = (row slot, column quad), 16-byte accesses, no per-element 64-bit divide
    const int q4 = hf >> 2, rpb = blockDim.x / q4;
    const int slot = threadIdx.x / q4, c4 = threadIdx.x - slot * q4;
    if (slot < rpb) {
      const float4 ar = __ldg(reinterpret_cast<const float4*>(a_r) + c4);
      const int k = (c4 * 4) / f;
      for (int64_t r = (int64_t)blockIdx.x * rpb + slot; r < rows; r += (int64_t)gridDim.x * rpb) {
        const float g = dAr[r * h + k];
        const float4 x = reinterpret_cast<const float4*>(recvH + r * hf)[c4];
        float4* o = reinterpret_cast<float4*>(dHt + r * hf) + c4;
        float4 v = *o;
        v.x += x.x + g * ar.x; v.y += x.y + g * ar.y; v.z += x.z + g * ar.z; v.w += x.w + g * ar.w;
        *o = v;
      }
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x)
      dAl[i] += recvAl[i];
    return;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n1 + n2; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n1) {
      const int64_t r = i / hf;
      const int c = (int)(i - r * hf);
      dHt[i] += recvH[i] + dAr[r * h + c / f] * __ldg(a_r + c);
    } else {
      dAl[i - n1] += recvAl[i - n1];
    }
  }
}

int grid_for(int64_t n, int per_block = 256) {
  const int64_t g = (n + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

size_t fl(int64_t n) { return align_up((size_t)std::max<int64_t>(n, 0) * sizeof(float)); }

int check_part(const gnncg_part_t* p, int h, int f) {
  GNNCG_REQUIRE(p && p->csr_local && p->csr_remote && p->csc_local && p->csc_remote && p->csr_local_sched &&
                    p->csr_remote_sched && p->csc_local_sched && p->csc_remote_sched,
                GNNCG_ERR_ARG, "gat_dist: null partition member");
  GNNCG_REQUIRE(p->nparts >= 1 && p->rank >= 0 && p->rank < p->nparts && p->num_local >= 0 &&
                    p->maxrows >= p->num_local,
                GNNCG_ERR_ARG, "gat_dist: bad partition (nparts %d rank %d num_local %lld maxrows %lld)", p->nparts,
                p->rank, (long long)p->num_local, (long long)p->maxrows);
  GNNCG_REQUIRE(p->csr_local->num_rows == p->num_local && p->csr_remote->num_rows == p->num_local &&
                    p->csc_local->num_rows == p->num_local &&
                    p->csc_remote->num_rows == (int64_t)p->nparts * p->maxrows,
                GNNCG_ERR_SHAPE, "gat_dist: index rows do not match the partition");
  GNNCG_REQUIRE(p->csr_local->num_edges == p->csc_local->num_edges &&
                    p->csr_remote->num_edges == p->csc_remote->num_edges,
                GNNCG_ERR_SHAPE, "gat_dist: csr / csc edge counts differ");
  GNNCG_REQUIRE(h >= 1 && h <= 32 && f >= 1, GNNCG_ERR_SHAPE, "gat_dist: bad heads / f");
  if (p->bounds) {
    GNNCG_REQUIRE(p->bounds[0] == 0 && (int64_t)(p->bounds[p->rank + 1] - p->bounds[p->rank]) == p->num_local,
                  GNNCG_ERR_ARG, "gat_dist: bounds disagree with num_local");
    for (int q = 0; q < p->nparts; ++q)
      GNNCG_REQUIRE(p->bounds[q + 1] >= p->bounds[q] && (int64_t)(p->bounds[q + 1] - p->bounds[q]) <= p->maxrows,
                    GNNCG_ERR_ARG, "gat_dist: block %d larger than maxrows", q);
  }
  return GNNCG_OK;
}

size_t gat_ws_need(const gnncg_part_t* p, int h, int f) {
  return std::max(std::max(gnncg_gat_workspace(p->csr_local_sched, nullptr, h, f),
                           gnncg_gat_workspace(p->csr_remote_sched, nullptr, h, f)),
                  std::max(gnncg_gat_workspace(nullptr, p->csc_local_sched, h, f),
                           gnncg_gat_workspace(nullptr, p->csc_remote_sched, h, f)));
}

}  // namespace
}  // namespace gnncg_b200

using namespace gnncg_b200;

struct gnncg_comm {
  ncclComm_t nc = nullptr;
  bool owned = false;
  int nranks = 1, rank = 0, device = 0;
  cudaStream_t cs = nullptr;  // collective stream (overlap with the caller's compute stream)
  cudaEvent_t ready = nullptr, done = nullptr;
};

namespace {
int comm_finish_init(gnncg_comm* c) {
  GNNCG_CUDA_TRY(cudaGetDevice(&c->device));
  GNNCG_CUDA_TRY(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
  GNNCG_CUDA_TRY(cudaEventCreateWithFlags(&c->ready, cudaEventDisableTiming));
  GNNCG_CUDA_TRY(cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming));
  return GNNCG_OK;
}

// caller stream -> collective stream
int fork_to_comm(gnncg_comm* c, cudaStream_t s) {
  GNNCG_CUDA_TRY(cudaEventRecord(c->ready, s));
  GNNCG_CUDA_TRY(cudaStreamWaitEvent(c->cs, c->ready, 0));
  return GNNCG_OK;
}
int join_from_comm(gnncg_comm* c, cudaStream_t s) {
  GNNCG_CUDA_TRY(cudaEventRecord(c->done, c->cs));
  GNNCG_CUDA_TRY(cudaStreamWaitEvent(s, c->done, 0));
  return GNNCG_OK;
}
}  // namespace

extern "C" {

int gnncg_comm_unique_id(void* id) {
  GNNCG_REQUIRE(id, GNNCG_ERR_ARG, "comm_unique_id: null output");
  GNNCG_NCCL_API();
  ncclUniqueId u;
  GNNCG_NCCL_TRY(nccl().GetUniqueId(&u));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &u, sizeof(u));
  return GNNCG_OK;
}

int gnncg_comm_init(gnncg_comm_t** out, int nranks, int rank, const void* id) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(out && id && nranks >= 1 && rank >= 0 && rank < nranks, GNNCG_ERR_ARG, "comm_init: bad argument");
  GNNCG_NCCL_API();
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  gnncg_comm* c = new gnncg_comm();
  c->owned = true;
  c->nranks = nranks;
  c->rank = rank;
  ncclResult_t r = nccl().CommInitRank(&c->nc, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(GNNCG_ERR_NCCL, "ncclCommInitRank(%d, %d): %s", nranks, rank, nccl().GetErrorString(r));
  }
  int rc = comm_finish_init(c);
  if (rc) {
    gnncg_comm_destroy(c);
    return rc;
  }
  *out = c;
  return GNNCG_OK;
}

int gnncg_comm_init_nccl(gnncg_comm_t** out, void* nc) {
  GNNCG_DEVICE_GUARD();
  GNNCG_REQUIRE(out && nc, GNNCG_ERR_ARG, "comm_init_nccl: bad argument");
  GNNCG_NCCL_API();
  gnncg_comm* c = new gnncg_comm();
  c->nc = static_cast<ncclComm_t>(nc);
  c->owned = false;
  ncclResult_t r1 = nccl().CommCount(c->nc, &c->nranks), r2 = nccl().CommUserRank(c->nc, &c->rank);
  if (r1 != ncclSuccess || r2 != ncclSuccess) {
    delete c;
    return fail(GNNCG_ERR_NCCL, "comm_init_nccl: not a valid ncclComm_t");
  }
  int rc = comm_finish_init(c);
  if (rc) {
    gnncg_comm_destroy(c);
    return rc;
  }
  *out = c;
  return GNNCG_OK;
}

int gnncg_comm_destroy(gnncg_comm_t* c) {
  if (!c) return GNNCG_OK;
  if (c->cs) cudaStreamSynchronize(c->cs);
  if (c->ready) cudaEventDestroy(c->ready);
  if (c->done) cudaEventDestroy(c->done);
  if (c->cs) cudaStreamDestroy(c->cs);
  int rc = GNNCG_OK;
  if (c->owned && c->nc && nccl().ok) {
    ncclResult_t r = nccl().CommDestroy(c->nc);
    if (r != ncclSuccess) rc = fail(GNNCG_ERR_NCCL, "ncclCommDestroy: %s", nccl().GetErrorString(r));
  }
  delete c;
  return rc;
}

int gnncg_comm_size(const gnncg_comm_t* c) { return c ? c->nranks : 0; }
int gnncg_comm_rank(const gnncg_comm_t* c) { return c ? c->rank : -1; }

int gnncg_comm_allgather(gnncg_comm_t* c, const float* send, float* recv, int64_t count, void* stream) {
  GNNCG_REQUIRE(c && count >= 0 && (count == 0 || (send && recv)), GNNCG_ERR_ARG, "comm_allgather: bad argument");
  if (count == 0) return GNNCG_OK;
  GNNCG_NCCL_TRY(nccl().AllGather(send, recv, (size_t)count, ncclFloat32, c->nc, as_stream(stream)));
  return GNNCG_OK;
}

int gnncg_comm_reduce_scatter(gnncg_comm_t* c, const float* send, float* recv, int64_t count, void* stream) {
  GNNCG_REQUIRE(c && count >= 0 && (count == 0 || (send && recv)), GNNCG_ERR_ARG,
                "comm_reduce_scatter: bad argument");
  if (count == 0) return GNNCG_OK;
  GNNCG_NCCL_TRY(nccl().ReduceScatter(send, recv, (size_t)count, ncclFloat32, ncclSum, c->nc, as_stream(stream)));
  return GNNCG_OK;
}

int gnncg_comm_allreduce(gnncg_comm_t* c, float* buf, int64_t count, void* stream) {
  GNNCG_REQUIRE(c && count >= 0 && (count == 0 || buf), GNNCG_ERR_ARG, "comm_allreduce: bad argument");
  if (count == 0) return GNNCG_OK;
  GNNCG_NCCL_TRY(nccl().AllReduce(buf, buf, (size_t)count, ncclFloat32, ncclSum, c->nc, as_stream(stream)));
  return GNNCG_OK;
}

size_t gnncg_gat_dist_workspace(const gnncg_part_t* p, int h, int f) {
  if (check_part(p, h, f)) return 0;
  const int64_t n = p->num_local, mr = p->maxrows, hf = (int64_t)h * f;
  const size_t fwd = fl(n * hf) + 2 * fl(n * h);
  const size_t bwd = fl(n * gnncg_gat_rec_stride(h)) + fl(mr * hf) + fl(mr * h);
  return align_up(gat_ws_need(p, h, f)) + std::max(fwd, bwd);
}

int gnncg_gat_fwd_dist(gnncg_comm_t* comm, const gnncg_part_t* p, int h, int f, float slope, float* Ht_all,
                       float* Al_all, const float* Ar, float* out, float* m, float* d, void* ws, size_t ws_bytes,
                       void* stream) {
  GNNCG_DEVICE_GUARD();
  int rc = check_part(p, h, f);
  if (rc) return rc;
  GNNCG_REQUIRE(Ht_all && Al_all && (p->num_local == 0 || (Ar && out && m && d)), GNNCG_ERR_ARG,
                "gat_fwd_dist: null pointer");
  GNNCG_REQUIRE(!comm || comm->nranks == p->nparts, GNNCG_ERR_ARG, "gat_fwd_dist: communicator has %d ranks, "
                "partition %d", comm ? comm->nranks : 0, p->nparts);
  const size_t need = gnncg_gat_dist_workspace(p, h, f);
  GNNCG_REQUIRE(ws && ws_bytes >= need, GNNCG_ERR_WORKSPACE, "gat_fwd_dist: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = as_stream(stream);
  const int64_t n = p->num_local, mr = p->maxrows, hf = (int64_t)h * f;
  const size_t gws = align_up(gat_ws_need(p, h, f));
  char* scratch = static_cast<char*>(ws) + gws;
  float* outL = reinterpret_cast<float*>(scratch);
  float* mL = reinterpret_cast<float*>(scratch + fl(n * hf));
  float* dL = reinterpret_cast<float*>(scratch + fl(n * hf) + fl(n * h));

  const bool gather = comm && p->nparts > 1;
  if (gather) {  // Ht || A_l of every rank, on the collective stream
    rc = fork_to_comm(comm, s);
    if (rc) return rc;
    GNNCG_NCCL_TRY(nccl().GroupStart());
    if (p->bounds) {  // only the owned rows of each block: one in-place broadcast per root
      for (int q = 0; q < p->nparts; ++q) {
        const size_t nq = (size_t)(p->bounds[q + 1] - p->bounds[q]);
        float* bh = Ht_all + (int64_t)q * mr * hf;
        float* ba = Al_all + (int64_t)q * mr * h;
        GNNCG_NCCL_TRY(nccl().Broadcast(bh, bh, nq * (size_t)hf, ncclFloat32, q, comm->nc, comm->cs));
        GNNCG_NCCL_TRY(nccl().Broadcast(ba, ba, nq * (size_t)h, ncclFloat32, q, comm->nc, comm->cs));
      }
    } else {
      GNNCG_NCCL_TRY(nccl().AllGather(Ht_all + p->rank * mr * hf, Ht_all, (size_t)(mr * hf), ncclFloat32, comm->nc,
                                      comm->cs));
      GNNCG_NCCL_TRY(nccl().AllGather(Al_all + p->rank * mr * h, Al_all, (size_t)(mr * h), ncclFloat32, comm->nc,
                                      comm->cs));
    }
    GNNCG_NCCL_TRY(nccl().GroupEnd());
  }
  if (n == 0) return gather ? join_from_comm(comm, s) : GNNCG_OK;
  const bool has_local = p->csr_local->num_edges > 0, has_remote = p->csr_remote->num_edges > 0;
  // K2 over the local-source edges while the tables land (straight into out when it is the only part)
  const bool merge = has_local && has_remote;
  if (has_local || !has_remote) {
    rc = gnncg_gat_fwd(p->csr_local, p->csr_local_sched, h, f, slope, Ht_all, Al_all, Ar, merge ? outL : out,
                       merge ? mL : m, merge ? dL : d, ws, gws, stream);
    if (rc) return rc;
  }
  if (gather) {
    rc = join_from_comm(comm, s);
    if (rc) return rc;
  }
  if (!has_remote) return GNNCG_OK;
  rc = gnncg_gat_fwd(p->csr_remote, p->csr_remote_sched, h, f, slope, Ht_all, Al_all, Ar, out, m, d, ws, gws, stream);
  if (rc) return rc;
  if (merge) {
    const int vw = (f % 4 == 0) ? 4 : (f % 2 == 0 ? 2 : 1);
    const int g = grid_for(n, 8);
    if (vw == 4) gat_merge2_kernel<4><<<g, 256, 0, s>>>(n, h, f, outL, mL, dL, out, m, d);
    else if (vw == 2) gat_merge2_kernel<2><<<g, 256, 0, s>>>(n, h, f, outL, mL, dL, out, m, d);
    else gat_merge2_kernel<1><<<g, 256, 0, s>>>(n, h, f, outL, mL, dL, out, m, d);
    GNNCG_LAUNCH_CHECK();
  }
  return GNNCG_OK;
}

int gnncg_gat_bwd_dist(gnncg_comm_t* comm, const gnncg_part_t* p, int h, int f, float slope, const float* Ht_all,
                       const float* Al_all, const float* Ar, const float* m, const float* d, const float* out,
                       const float* dOut, const float* a_l, const float* a_r, float* dHt, float* dAl, float* dAr,
                       float* dHt_send, float* dAl_send, void* ws, size_t ws_bytes, void* stream) {
  GNNCG_DEVICE_GUARD();
  int rc = check_part(p, h, f);
  if (rc) return rc;
  GNNCG_REQUIRE(gnncg_gat_fast_supported(h, f), GNNCG_ERR_UNSUPPORTED,
                "gat_bwd_dist: heads=%d f=%d outside the fused backward's shapes", h, f);
  GNNCG_REQUIRE(Ht_all && Al_all && a_l && a_r && dHt_send && dAl_send &&
                    (p->num_local == 0 || (Ar && m && d && out && dOut && dHt && dAl && dAr)),
                GNNCG_ERR_ARG, "gat_bwd_dist: null pointer");
  GNNCG_REQUIRE(!comm || comm->nranks == p->nparts, GNNCG_ERR_ARG, "gat_bwd_dist: communicator has %d ranks, "
                "partition %d", comm ? comm->nranks : 0, p->nparts);
  const size_t need = gnncg_gat_dist_workspace(p, h, f);
  GNNCG_REQUIRE(ws && ws_bytes >= need, GNNCG_ERR_WORKSPACE, "gat_bwd_dist: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = as_stream(stream);
  const int64_t n = p->num_local, mr = p->maxrows, hf = (int64_t)h * f;
  const size_t gws = align_up(gat_ws_need(p, h, f));
  char* scratch = static_cast<char*>(ws) + gws;
  const int rs = gnncg_gat_rec_stride(h);
  float* rec = reinterpret_cast<float*>(scratch);
  float* recvH = reinterpret_cast<float*>(scratch + fl(n * rs));
  float* recvAl = reinterpret_cast<float*>(scratch + fl(n * rs) + fl(mr * hf));

  if (n > 0) {
    rc = gnncg_gat_bwd_prep(n, h, f, dOut, out, Ar, m, d, rec, stream);
    if (rc) return rc;
  }
  const bool multi = p->nparts > 1;
  // 1. the partials other ranks own: K4f over the remote-source edges (every padded row written)
  if (multi) {
    rc = gat_bwd_src_fused_pass(p->csc_remote, p->csc_remote_sched, h, f, slope, n, Ht_all, Al_all, rec, dOut, a_l,
                                a_r, dHt_send, dAl_send, dAr, /*zero_dar=*/true, ws, gws, s);
    if (rc) return rc;
  }
  // 2. their reduce-scatter on the collective stream ...
  const bool scatter = comm && multi;
  if (scatter) {
    rc = fork_to_comm(comm, s);
    if (rc) return rc;
    GNNCG_NCCL_TRY(nccl().GroupStart());
    if (p->bounds) {  // block q's partials summed onto rank q, owned rows only
      for (int q = 0; q < p->nparts; ++q) {
        const size_t nq = (size_t)(p->bounds[q + 1] - p->bounds[q]);
        GNNCG_NCCL_TRY(nccl().Reduce(dHt_send + (int64_t)q * mr * hf, recvH, nq * (size_t)hf, ncclFloat32, ncclSum, q,
                                     comm->nc, comm->cs));
        GNNCG_NCCL_TRY(nccl().Reduce(dAl_send + (int64_t)q * mr * h, recvAl, nq * (size_t)h, ncclFloat32, ncclSum, q,
                                     comm->nc, comm->cs));
      }
    } else {
      GNNCG_NCCL_TRY(
          nccl().ReduceScatter(dHt_send, recvH, (size_t)(mr * hf), ncclFloat32, ncclSum, comm->nc, comm->cs));
      GNNCG_NCCL_TRY(
          nccl().ReduceScatter(dAl_send, recvAl, (size_t)(mr * h), ncclFloat32, ncclSum, comm->nc, comm->cs));
    }
    GNNCG_NCCL_TRY(nccl().GroupEnd());
  }
  // 3. ... while K4f walks the local-source edges (own rows of the tables, rebased)
  if (n > 0) {
    rc = gat_bwd_src_fused_pass(p->csc_local, p->csc_local_sched, h, f, slope, n, Ht_all + p->rank * mr * hf,
                                Al_all + p->rank * mr * h, rec, dOut, a_l, a_r, dHt, dAl, dAr, /*zero_dar=*/!multi, ws,
                                gws, s);
    if (rc) return rc;
  }
  if (scatter) {
    rc = join_from_comm(comm, s);
    if (rc) return rc;
  }
  if (n == 0) return GNNCG_OK;
  // 4. dHt = own + received + dA_r (x) a_r ; dAl = own + received
  if (scatter) {
    gat_dist_combine_kernel<<<grid_for(n * (hf + h)), 256, 0, s>>>(n, h, f, recvH, recvAl, dAr, a_r, dHt, dAl);
    GNNCG_LAUNCH_CHECK();
    return GNNCG_OK;
  }
  return gat_lp_dar(n, h, f, dAr, a_r, dHt, s);
}

}  // extern "C"
