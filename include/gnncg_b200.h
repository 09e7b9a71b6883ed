/* SPDX-License-Identifier: Apache-2.0
 *
 * gnncg_b200.h -- C ABI of the B200-native (sm_100a) fused GNN layer path.
 *
 * This is the drop-in boundary for the reference's fused-layer path.  The
 * reference ("gnncg", /root/reference/proj) specifies -- but does not ship -- an
 * executor that runs the fused GAT / EdgeConv / GMMConv graph regions over its
 * dual index.  Every entry point below replaces one operation
 * of that executor or of the graph/tensor layer it sits on; the replaced
 * interface is cited (file:line) beside each declaration.
 *
 * Conventions (identical to the reference's data model):
 *   - an index is gnncg::AdjIndex (graph.hpp:19-29) split to SoA:
 *       off[rows+1] = AdjIndex::offsets, nbr[E] = entries[i].vertex,
 *       eid[E] = entries[i].edge; rows are sorted by edge id (graph.hpp:26).
 *   - tensors are row-major gnncg::Tensor<float> (tensor.hpp:20-35); multi-head
 *     features are flattened head-major, cols = h*f, column j -> head j/f
 *     (tensor.hpp:17-19,99-121).
 *   - LeakyReLU(z) = z > 0 ? z : slope*z (tensor.hpp:75), slope default 0.2.
 *   - every pointer argument is DEVICE memory unless the name ends in _host.
 *   - calls are asynchronous on the given stream (a cudaStream_t passed as
 *     void*; NULL = legacy default stream).  The library never allocates device
 *     memory inside compute calls; scratch comes from the caller's workspace,
 *     sized by the matching *_workspace() query.
 *   - errors: the return value is a gnncg_status; gnncg_last_error() returns a
 *     thread-local message.  Shape errors correspond to the reference's
 *     TensorError (tensor.hpp:13-15), range errors to GraphError (graph.hpp:14-16).
 *     There is no CPU fallback: without an sm_100 device every compute call
 *     returns GNNCG_ERR_NO_DEVICE.
 *
 * Row partitioning (multi-GPU): a call may process a contiguous block of
 * destination rows.  "Destination-side" tensors (indexed by an index row of
 * csr_dst: out, m, d, A_r, dOut, c, dA_r) are LOCAL (row 0 = first row of the
 * block); "source-side" tensors (indexed by a neighbour id of csr_dst: Ht, A_l)
 * are GLOBAL.  A single-GPU caller simply passes the whole graph.
 */
#ifndef GNNCG_B200_H_
#define GNNCG_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum gnncg_status {
  GNNCG_OK = 0,
  GNNCG_ERR_SHAPE = 1,       /* TensorError: shape / width mismatch (tensor.hpp:13-15) */
  GNNCG_ERR_RANGE = 2,       /* GraphError: endpoint out of range (graph.cpp:37-39) */
  GNNCG_ERR_NO_DEVICE = 3,   /* no sm_100 device visible: no CPU fallback exists */
  GNNCG_ERR_CUDA = 4,        /* CUDA runtime / launch failure */
  GNNCG_ERR_WORKSPACE = 5,   /* caller workspace smaller than the *_workspace() query */
  GNNCG_ERR_UNSUPPORTED = 6, /* shape outside the compiled kernel variants */
  GNNCG_ERR_ARG = 7,         /* null pointer / invalid argument */
  GNNCG_ERR_NCCL = 8         /* NCCL library missing or a collective failed */
} gnncg_status;

/* One adjacency index (AdjIndex, graph.hpp:19-29), possibly a row block of it. */
typedef struct gnncg_index {
  int64_t num_rows;    /* rows processed (block length; V for a whole index) */
  int64_t num_edges;   /* off[num_rows] - off[0]; off[0] must be 0 (rebased block) */
  const uint64_t* off; /* num_rows + 1 */
  const uint32_t* nbr; /* AdjEntry::vertex */
  const uint32_t* eid; /* AdjEntry::edge; may be NULL where unused */
} gnncg_index_t;

/* Edge-balance schedule over one index: "unified thread mapping" work items
 * (one warp each).  Rows with more than `chunk` edges are split into several
 * items whose partial results are merged deterministically in chunk order --
 * the reference's ReductionBuffer contract applied to the
 * fused region, which the online-softmax merge makes legal for GAT
 * (cf. SPEC.md:267-268).  Built on the host by gnncg_sched_build_host(). */
typedef struct gnncg_sched {
  int64_t num_items;       /* total work items */
  int64_t num_split_items; /* items [0, num_split_items) belong to split rows */
  int64_t num_split_rows;
  int32_t chunk;           /* max edges per item */
  int32_t reserved;
  const uint32_t* items;       /* 2*num_items: (row, chunk index) pairs */
  const uint32_t* split_rows;  /* num_split_rows row ids */
  const uint32_t* split_first; /* num_split_rows+1 item offsets into [0, num_split_items) */
  /* Optional L2 hint (NULL / 0 = none): HOST prefix sums of how often each row of the table the
   * kernel GATHERS is read, i.e. the offsets of the other index (csc_src's for a csr_dst schedule:
   * K2 gathers source rows; csr_dst's for a csc_src schedule: K4f gathers destination rows), and
   * their row count.  With gnncg_l2_persist() on, the fp32 fused kernels mark the contiguous row
   * range carrying the most gathers as L2-persisting (gnncg_hot_window_host).  Caller-owned and
 * not modified while in use: the window is computed once per (gather_off, gather_rows, size). */
  const uint64_t* gather_off;
  int64_t gather_rows;
} gnncg_sched_t;

/* ---------------------------------------------------------------- runtime */
const char* gnncg_last_error(void);
const char* gnncg_version(void);
/* GNNCG_OK iff an sm_100 (B200) device is current. */
int gnncg_device_check(void);
/* Number of kernels this library has launched in the process (instrumentation). */
uint64_t gnncg_launch_count(void);
/* Cost counters (instrumentation; "measured flops / io_units == predicted").
 * `counters` = a zeroed DEVICE array of 10 uint64 (NULL turns counting off).  While set, every
 * GAT kernel adds the edges each work item walks and the rows it completes to its pair
 * (edges, rows):
 *   [0,1] K2 (fwd, fp32 or bf16)  [2,3] K3  [4,5] K4  [6,7] K4f (fused fast backward)
 *   [8,9] the attention LPs (gnncg_gat_transform's epilogue / gnncg_gat_attn_dots): rows, calls.
 * The sums equal (|E|, rows) per call iff every edge was aggregated exactly once and every row
 * written once; the flops / io units follow from each kernel's fixed per-edge and per-row work
 * (paper_2110_09524_b200/cost.py).  Process-wide; not for concurrent measurement. */
int gnncg_cost_counters(uint64_t* counters);
/* L2 residency for the gathered tables (opt-in, process-wide).  Sets the device's persisting-L2
 * set-aside to min(bytes, cudaDevAttrMaxPersistingL2CacheSize) (0 turns it off and resets the
 * persisting lines); *granted_host (may be NULL) receives the size set.  While on, the fp32
 * fused GAT kernels (K2, K4f) launch with an access-policy window over the hottest rows of the
 * table they gather (schedules carrying gather_off): those rows stay in L2, the rest streams.
 * The window is used only when its rows carry at least twice their share of the reads (row ids
 * clustered by degree, e.g. after DeviceGraph.relabel(degree_order())); otherwise the launch is
 * plain.  Results do not change (cache policy only). */
int gnncg_l2_persist(size_t bytes, size_t* granted_host);
/* The window: the start row b maximising off[b+n] - off[b] (the gathers of rows [b, b+n)) over
 * 0 <= b <= num_rows - n, lowest b on ties; n is clamped to num_rows. */
int gnncg_hot_window_host(int64_t num_rows, const uint64_t* off_host, int64_t n, int64_t* begin_host);

/* ------------------------------------------------------- graph store (K9)
 * Replaces build_index (graph.cpp:14-28) and the Graph ctor (graph.cpp:32-45).
 * Counting sort by key vertex, stable in edge id -> bit-identical to the
 * reference's AdjIndex.  key/other/off/nbr/eid are device arrays.  Returns
 * GNNCG_ERR_RANGE if any endpoint >= V (the reference's GraphError). */
size_t gnncg_csr_build_workspace(int64_t num_vertices, int64_t num_edges);
int gnncg_csr_build(int64_t num_vertices, int64_t num_edges, const uint32_t* key, const uint32_t* other,
                    uint64_t* off, uint32_t* nbr, uint32_t* eid, void* workspace, size_t workspace_bytes,
                    void* stream);
/* Rectangular variant for rank-local indexes (multi-GPU, dist.py): keys are rows
 * [0, num_rows) of a destination block, neighbour ids range over [0, num_other) (the
 * padded all-gather layout of every rank's sources).  Same sort and error contract;
 * gnncg_csr_build(V, ...) == gnncg_csr_build_rect(V, V, ...). */
int gnncg_csr_build_rect(int64_t num_rows, int64_t num_other, int64_t num_edges, const uint32_t* key,
                         const uint32_t* other, uint64_t* off, uint32_t* nbr, uint32_t* eid, void* workspace,
                         size_t workspace_bytes, void* stream);

/* degree_stats (graph.cpp:47-57) over a device index: out_host[0] = max degree
 * of `idx` (blocking call; stream is synchronised). */
int gnncg_max_degree(const gnncg_index_t* idx, uint64_t* max_degree_host, void* stream);

/* Row-block partitioner (new): P contiguous row blocks with
 * balanced edge counts, bound[p] = lower_bound(off, ceil(p*E/P)), bound[P] = V.
 * off_host/bound_host are host arrays. */
int gnncg_partition_rows(int64_t num_rows, const uint64_t* off_host, int32_t parts, uint64_t* bound_host);
/* Cost-balanced variant: row v costs its edges plus row_weight (the per-row work of a layer in
 * edge units: the row's share of the transform / gradient GEMMs, records, per-item overheads),
 *   cost(v) = off[v] + row_weight * v,  bound[p] = lower_bound(cost, ceil(p * cost(V) / P)).
 * row_weight = 0 is gnncg_partition_rows.  Edge-balanced blocks of a power-law graph give the
 * rank with the low-degree tail ~45x the rows of the hub rank and ~2x its step time (C5, P = 8,
 * scripts/emulate_ranks.py). */
int gnncg_partition_rows_weighted(int64_t num_rows, const uint64_t* off_host, int32_t parts, uint64_t row_weight,
                                  uint64_t* bound_host);

/* Deterministic Chung-Lu edge generator (device): edge e draws its destination
 * and source independently from the integer weight CDF `cdf` (device, V entries,
 * inclusive prefix sums of positive weights), using the counter-based hash
 * splitmix64(seed, e).  Same edge list for the same (cdf, seed) on any device. */
int gnncg_gen_chung_lu(int64_t num_vertices, int64_t num_edges, const uint64_t* cdf, uint64_t seed, uint32_t* src,
                       uint32_t* dst, void* stream);

/* Per-rank generation of the same edge list (multi-GPU: every rank keeps only its own
 * destination rows).  gnncg_gen_chung_lu_degrees writes the in-degree of every
 * vertex (u32, device) -- the offsets the row partitioner splits; gnncg_gen_chung_lu_rows
 * writes, in edge-id order, the edges whose destination lies in [row_begin, row_end):
 * src/dst hold off[row_end] - off[row_begin] entries (workspace sized by
 * gnncg_gen_chung_lu_rows_workspace).  Together they equal filtering gnncg_gen_chung_lu's
 * list by destination, without materialising it. */
int gnncg_gen_chung_lu_degrees(int64_t num_vertices, int64_t num_edges, const uint64_t* cdf, uint64_t seed,
                               uint32_t* in_deg, void* stream);
size_t gnncg_gen_chung_lu_rows_workspace(int64_t num_edges);
int gnncg_gen_chung_lu_rows(int64_t num_vertices, int64_t num_edges, const uint64_t* cdf, uint64_t seed,
                            int64_t row_begin, int64_t row_end, uint32_t* src, uint32_t* dst, void* workspace,
                            size_t workspace_bytes, void* stream);

/* Schedule construction on the host from a host copy of the offsets.
 * First call with items_host == NULL to get the counts, then with arrays sized
 * 2*num_items, num_split_rows, num_split_rows+1. */
int gnncg_sched_build_host(int64_t num_rows, const uint64_t* off_host, int32_t chunk, int64_t* num_items,
                           int64_t* num_split_items, int64_t* num_split_rows, uint32_t* items_host,
                           uint32_t* split_rows_host, uint32_t* split_first_host);

/* ------------------------------------------------- dense transforms (K1/K5)
 * C[M,N] = op(A)[M,K] * op(B)[K,N], fp32 in / fp32 accumulate / fp32 out.
 * trans_a = 0: A is M x K (lda >= K);  trans_a = 1: A is K x M (lda >= M).
 * trans_b = 0: B is K x N (ldb >= N);  trans_b = 1: B is N x K (ldb >= K).
 * (0,0) = matmul (tensor.cpp:8-24); (0,1) = matmul_nt (tensor.cpp:26-42);
 * (1,0) = matmul_tn (tensor.cpp:44-60).  Deterministic (fixed-order split-K). */
size_t gnncg_gemm_workspace(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K);
int gnncg_gemm(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
               const float* B, int64_t ldb, float* C, int64_t ldc, void* workspace, size_t workspace_bytes,
               void* stream);

/* ------------------------------------------------------------------ GAT
 * Reorganized attention LPs:
 *   A_l[v,k] = <Ht[v,k,:], a_l[k,:]>, A_r[v,k] = <Ht[v,k,:], a_r[k,:]>. */
int gnncg_gat_attn_dots(int64_t num_rows, int heads, int f, const float* Ht, const float* a_l, const float* a_r,
                        float* Al, float* Ar, void* stream);

/* K1 with its epilogue: Ht = H W (H is M x K with row stride ldh, W is K x heads*f, Ht dense)
 * AND the reorganized LPs A_l = Ht . a_l, A_r = Ht . a_r computed by the tensor-core GEMM's
 * epilogue from the accumulator it already holds (SURVEY K1 "attn-dot epilogue"; bitwise equal
 * to gnncg_gemm + gnncg_gat_attn_dots).  Shapes outside the fused kernel (f % 32 != 0, split-K)
 * run those two calls instead.  Workspace: gnncg_gemm_workspace(0, 0, M, heads*f, K). */
int gnncg_gat_transform(int64_t M, int64_t K, int heads, int f, const float* H, int64_t ldh, const float* W,
                        float* Ht, const float* a_l, const float* a_r, float* Al, float* Ar, void* workspace,
                        size_t workspace_bytes, void* stream);

/* Scratch for the split-row partials of all GAT kernels over these schedules, plus the work
 * counter K2 / K4f pull their items from (zeroed by the call itself; a smaller workspace that
 * still holds the partials makes them walk the items with a fixed stride instead).  One
 * workspace must not be shared by GAT calls running concurrently on different streams. */
size_t gnncg_gat_workspace(const gnncg_sched_t* dst_sched, const gnncg_sched_t* src_sched, int heads, int f);

/* K2: the fused region Scatter(u_add_v) -> ApplyEdge(LeakyReLU) ->
 * ReduceScatter(edge-softmax RS1/RS2) -> Aggregate(sum) in ONE kernel
 * (PAPER.md:316-319,555-558), vertex-balanced with the
 * edge-balance split of `sched`.  Stashes only m, d (V x h).
 *   out[v,k,:] = sum_e softmax_v(LReLU(A_l[u,k] + A_r[v,k])) * Ht[u,k,:]
 * Empty rows: out = 0, m = d = 0. */
int gnncg_gat_fwd(const gnncg_index_t* csr_dst, const gnncg_sched_t* sched, int heads, int f, float slope,
                  const float* Ht, const float* Al, const float* Ar, float* out, float* m, float* d,
                  void* workspace, size_t workspace_bytes, void* stream);

/* K3: backward pass 1 over csr_dst (derive_backward + plan_recompute,
 * SPEC.md:187-195,273-281,352-360): edge values recomputed from (A_l, A_r, m, d);
 *   c[v,k]   = sum_e alpha_e <dOut[v,k,:], Ht[u,k,:]>
 *   dA_r[v,k] = sum_e LReLU'(z_e) alpha_e (dalpha_e - c[v,k]) */
int gnncg_gat_bwd_dst(const gnncg_index_t* csr_dst, const gnncg_sched_t* sched, int heads, int f, float slope,
                      const float* Ht, const float* Al, const float* Ar, const float* m, const float* d,
                      const float* dOut, float* c, float* dAr, void* workspace, size_t workspace_bytes,
                      void* stream);

/* K4: backward pass 2 over csc_src (Scatter backward = Gather over out-edges,
 * PAPER.md:638-649).  Rows are GLOBAL source ids u; neighbours are LOCAL
 * destination rows of the block [row_base, row_base + num_local_rows).
 *   dA_l[u,k] = sum_e LReLU'(z_e) alpha_e (dalpha_e - c[v,k])
 *   dHt[u,:]  = sum_e alpha_e dOut[v,:] + dA_l[u] (x) a_l + dA_r[u] (x) a_r
 * (the dA_r term only for u inside the local block).  In a multi-GPU run the
 * outputs are partial sums to be reduce-scattered (they are linear). */
int gnncg_gat_bwd_src(const gnncg_index_t* csc_src, const gnncg_sched_t* sched, int heads, int f, float slope,
                      int64_t row_base, int64_t num_local_rows, const float* Ht, const float* Al, const float* Ar,
                      const float* m, const float* d, const float* c, const float* dOut, const float* dAr,
                      const float* a_l, const float* a_r, float* dHt, float* dAl, void* workspace,
                      size_t workspace_bytes, void* stream);

/* Fast mode (lock-free atomic accumulation, tolerance-tested): K3 folded
 * into K4.  gnncg_gat_bwd_prep builds, per destination row v and head k, the record
 * float4 {A_r[v,k], lse[v,k] = m + log d, c[v,k] = <dOut[v,k,:], out[v,k,:]>, 0}
 * (row stride gnncg_gat_rec_stride(heads) = 4 heads floats; c = sum_e alpha_e dalpha_e by the
 * softmax-backward identity, so no pass over csr_dst is needed).  One pass over
 * csc_src then produces dHt (including both LP terms), dA_l, and dA_r (zeroed and
 * accumulated with global reductions: order-nondeterministic in the last bits).
 * Supported when gnncg_gat_fast_supported(heads, f) != 0. */
int gnncg_gat_fast_supported(int heads, int f);
int gnncg_gat_rec_stride(int heads);
int gnncg_gat_bwd_prep(int64_t num_rows, int heads, int f, const float* dOut, const float* out, const float* Ar,
                       const float* m, const float* d, float* dst_rec, void* stream);
int gnncg_gat_bwd_src_fused(const gnncg_index_t* csc_src, const gnncg_sched_t* sched, int heads, int f, float slope,
                            int64_t row_base, int64_t num_local_rows, const float* Ht, const float* Al,
                            const float* dst_rec, const float* dOut, const float* a_l, const float* a_r, float* dHt,
                            float* dAl, float* dAr, void* workspace, size_t workspace_bytes, void* stream);

/* bf16 gather tables (the north star's "bf16 features" option, with a stated looser bound):
 * K2 gathers Ht[u] rows and K4f gathers dOut[v] rows from bf16 copies (round to nearest even);
 * logits, records, every accumulation and every output stay fp32.  Half the gathered bytes
 * per edge.  Consistency of the recompute backward: K4f takes the own row from the same bf16
 * Ht the forward aggregated, and gnncg_gat_bwd_prep_bf16 forms c = <bf16(dOut), out> while it
 * writes the bf16 dOut table, so sum_e alpha_e dalpha_e = c[v] holds as in fp32 mode.
 * Same semantics and workspaces as gnncg_gat_fwd / gnncg_gat_bwd_prep /
 * gnncg_gat_bwd_src_fused; supported when gnncg_gat_bf16_supported(heads, f) != 0
 * (f % 4 == 0, heads * f <= 512).  Replaces the same spec ops. */
int gnncg_gat_bf16_supported(int heads, int f);
int gnncg_pack_bf16(int64_t n, const float* src, uint16_t* dst, void* stream);
int gnncg_gat_fwd_bf16(const gnncg_index_t* csr_dst, const gnncg_sched_t* sched, int heads, int f, float slope,
                       const uint16_t* Ht_bf16, const float* Al, const float* Ar, float* out, float* m, float* d,
                       void* workspace, size_t workspace_bytes, void* stream);
int gnncg_gat_bwd_prep_bf16(int64_t num_rows, int heads, int f, const float* dOut, const float* out,
                            const float* Ar, const float* m, const float* d, float* dst_rec, uint16_t* dOut_bf16,
                            void* stream);
int gnncg_gat_bwd_src_fused_bf16(const gnncg_index_t* csc_src, const gnncg_sched_t* sched, int heads, int f,
                                 float slope, int64_t row_base, int64_t num_local_rows, const uint16_t* Ht_bf16,
                                 const float* Al, const float* dst_rec, const uint16_t* dOut_bf16, const float* a_l,
                                 const float* a_r, float* dHt, float* dAl, float* dAr, void* workspace,
                                 size_t workspace_bytes, void* stream);

/* da_l[k,:] = sum_v dA_l[v,k] Ht[v,k,:] ; da_r likewise (LP parameter grads). */
size_t gnncg_gat_attn_grad_workspace(int64_t num_rows, int heads, int f);
int gnncg_gat_attn_grad(int64_t num_rows, int heads, int f, const float* Ht, const float* dAl, const float* dAr,
                        float* da_l, float* da_r, void* workspace, size_t workspace_bytes, void* stream);

/* -------------------------------------------------------------- EdgeConv
 * K6 (reorganized per SPEC.md:261): Th = H Theta, Ph = H Phi
 * precomputed (packed as Y = [Th | Ph], row stride ldy).
 *   out[v,c] = max_e ((Th[u,c] - Th[v,c]) + Ph[v,c])  evaluated in fp32 RN
 *   argmax[v,c] = edge id of the lowest-eid maximiser, or
 *   0xFFFFFFFF with out = 0 for an empty row.  Bit-exact.
 * Th is indexed by global ids, Ph / out / argmax by local rows. */
int gnncg_edgeconv_fwd(const gnncg_index_t* csr_dst, int channels, int64_t row_base, const float* Th,
                       int64_t ld_th, const float* Ph, int64_t ld_ph, float* out, uint32_t* argmax, void* stream);

/* K7: Gather(max) backward by argmax routing, atomic-free
 * (inverse-argmax gather over csc_src, needs csc_src.eid):
 *   dTh[u,c] = sum_{(v,e) in out(u), argmax[v,c]==e} g[v,c] - [deg_in(u)>0] g[u,c]
 *   dPh[u,c] = [deg_in(u)>0] g[u,c] */
int gnncg_edgeconv_bwd(const gnncg_index_t* csc_src, const gnncg_index_t* csr_dst, int channels,
                       const uint32_t* argmax, const float* grad, float* dTh, int64_t ld_dth, float* dPh,
                       int64_t ld_dph, void* stream);

/* --------------------------------------------------------------- GMMConv
 * K8: Y = H [W | P_l | P_r] packed, row stride
 * ldy = K*f + 2r: hW = Y[:, :K*f], pl = Y[:, K*f:K*f+r], pr = Y[:, K*f+r:].
 *   w_k(m) = exp(-1/2 sum_d (m_d - mu_kd)^2 sinv_kd^2),  m = pl[u] + pr[v]
 *   out[v,:] = (1/K) sum_e sum_k w_k hW[u,k,:] */
int gnncg_gmm_fwd(const gnncg_index_t* csr_dst, int kernels, int r, int f, const float* Y, int64_t ldy,
                  const float* mu, const float* sinv, float* out, void* stream);

size_t gnncg_gmm_bwd_workspace(const gnncg_index_t* csr_dst, int kernels, int r);
/* Backward: dY (same packing as Y) and parameter grads dmu, dsinv (K x r).
 * pass 1 over csr_dst -> d pr, dmu, dsinv ; pass 2 over csc_src -> d hW, d pl. */
int gnncg_gmm_bwd(const gnncg_index_t* csr_dst, const gnncg_index_t* csc_src, int kernels, int r, int f,
                  const float* Y, int64_t ldy, const float* mu, const float* sinv, const float* dOut, float* dY,
                  float* dmu, float* dsinv, void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------ GCN (weighted Aggregate)
 * SURVEY §8f rank 3; the spec's gcn model:
 *   [ApplyVertex(W), Scatter(copy_u), ApplyEdge(x e_uv), Gather(sum), ApplyVertex(+b, sigma)]
 * One kernel over `idx` (csr_dst forward, csc_src for the transpose in backward):
 *   Y[r,:] = act(bias + sum_{i in row r} w[eid_i] X[nbr_i,:])
 * edge_w is indexed by edge id (NULL = all ones; non-NULL needs idx->eid); bias may be
 * NULL; relu != 0 applies max(0,.).  Rows of idx are local (Y has idx->num_rows rows),
 * neighbours global.  Deterministic (fixed-order split-row merge).  The workspace holds the
 * split-row partials and a work counter: one workspace per concurrently running call. */
size_t gnncg_spmm_workspace(const gnncg_sched_t* sched, int cols);
int gnncg_spmm(const gnncg_index_t* idx, const gnncg_sched_t* sched, int cols, const float* edge_w, const float* X,
               const float* bias, int relu, float* Y, void* workspace, size_t workspace_bytes, void* stream);
/* Backward of the epilogue: dZ = dOut * [out > 0] (relu) or dOut; dbias (if non-NULL) =
 * column sums of dZ (fixed order). */
size_t gnncg_relu_bwd_workspace(int cols);
int gnncg_relu_bwd(int64_t rows, int cols, const float* dOut, const float* out, int relu, float* dZ, float* dbias,
                   void* workspace, size_t workspace_bytes, void* stream);
/* Symmetric GCN normalisation by edge id:
 *   w[e] = 1 / sqrt(max(1, deg_in(dst e)) * max(1, deg_out(src e))) */
int gnncg_gcn_norm(int64_t num_edges, const uint32_t* edge_src, const uint32_t* edge_dst,
                   const gnncg_index_t* csr_dst, const gnncg_index_t* csc_src, float* w, void* stream);

/* ------------------------------------------------ multi-GPU
 * The reference's executor is single-process; north_star partitions the graph's destination
 * rows over P GPUs (one process each) with one all-gather per layer forward and a
 * reduce-scatter per layer backward.  These entry points replace the spec's run_forward /
 * run_backward for one rank of such a run.
 *
 * Communicator: a thin handle over an NCCL communicator plus a private collective stream.
 * NCCL is resolved at run time (dlopen of libnccl.so.2: the copy already loaded in the
 * process if any, e.g. torch's, else the system one), so this library has no link-time
 * NCCL dependency; GNNCG_ERR_NCCL if it is absent.  Either create one from an NCCL unique
 * id (rank 0 calls gnncg_comm_unique_id and the caller distributes the 128 bytes), or wrap a
 * caller-owned ncclComm_t (gnncg_comm_init_nccl; not destroyed by gnncg_comm_destroy). */
typedef struct gnncg_comm gnncg_comm_t;
int gnncg_comm_unique_id(void* id_128_bytes_host);
int gnncg_comm_init(gnncg_comm_t** comm_out_host, int nranks, int rank, const void* id_128_bytes_host);
int gnncg_comm_init_nccl(gnncg_comm_t** comm_out_host, void* nccl_comm);
int gnncg_comm_destroy(gnncg_comm_t* comm);
int gnncg_comm_size(const gnncg_comm_t* comm);
int gnncg_comm_rank(const gnncg_comm_t* comm);
/* fp32 collectives on `stream` (the caller's; ordered with its other work):
 * recv[P*count] = concat over ranks of send[count] (send may be recv + rank*count: in place);
 * recv[count] = sum over ranks of send[rank*count : (rank+1)*count];  buf[count] summed in place. */
int gnncg_comm_allgather(gnncg_comm_t* comm, const float* send, float* recv, int64_t count, void* stream);
int gnncg_comm_reduce_scatter(gnncg_comm_t* comm, const float* send, float* recv, int64_t count, void* stream);
int gnncg_comm_allreduce(gnncg_comm_t* comm, float* buf, int64_t count, void* stream);

/* One rank's share of a destination-row partition (dist.py builds it):
 *   rows [r_p, r_p + num_local) of csr_dst are owned; every source-side table (Ht, A_l) lives
 *   in the PADDED all-gather layout: rank q's rows at [q*maxrows, q*maxrows + n_q).
 *   The rank's in-edges are split by the owner of their source:
 *     csr_local  / csc_local  -- sources in this rank's block (available before the all-gather);
 *     csr_remote / csc_remote -- sources of other ranks.
 *   csr_*: rows = num_local destinations, neighbour = padded source id.
 *   csc_local: rows = num_local own sources (row r = padded id rank*maxrows + r),
 *              neighbour = local destination row.
 *   csc_remote: rows = nparts*maxrows padded sources (this rank's block empty),
 *              neighbour = local destination row.
 * Each index carries its edge-balance schedule (gnncg_sched_build_host). */
typedef struct gnncg_part {
  int64_t num_local;
  int64_t maxrows;
  int32_t nparts;
  int32_t rank;
  const gnncg_index_t* csr_local;
  const gnncg_sched_t* csr_local_sched;
  const gnncg_index_t* csr_remote;
  const gnncg_sched_t* csr_remote_sched;
  const gnncg_index_t* csc_local;
  const gnncg_sched_t* csc_local_sched;
  const gnncg_index_t* csc_remote;
  const gnncg_sched_t* csc_remote_sched;
  /* Optional HOST row bounds of all ranks (nparts + 1 entries; NULL = unknown).  With them the
   * collectives move only the rows each rank owns -- grouped ncclBroadcast / ncclReduce per
   * block into the padded layout -- instead of nparts x maxrows rows (ncclAllGather /
   * ncclReduceScatter over the padding): at C5, P = 8, 10M instead of 20M rows per layer. */
  const uint64_t* bounds;
} gnncg_part_t;

size_t gnncg_gat_dist_workspace(const gnncg_part_t* part, int heads, int f);

/* Partitioned K2 (the fused GAT region forward of one rank):
 *   the caller has written its own rows of Ht_all (nparts*maxrows x h*f) and Al_all
 *   (nparts*maxrows x h) at block `rank` (gnncg_gat_transform into those rows);
 *   the all-gather of both tables runs on the communicator's stream while K2 aggregates the
 *   local-source edges on `stream`; K2 then aggregates the remote-source edges and the two
 *   online-softmax partials are merged:  m = max(m1, m2), d = d1 e^(m1-m) + d2 e^(m2-m),
 *   out = (d1 e^(m1-m) out1 + d2 e^(m2-m) out2) / d  (an empty part contributes nothing).
 *   out / m / d / Ar: num_local rows.  comm == NULL: the tables are already complete (no
 *   collective; e.g. a caller that gathered them itself). */
int gnncg_gat_fwd_dist(gnncg_comm_t* comm, const gnncg_part_t* part, int heads, int f, float slope, float* Ht_all,
                       float* Al_all, const float* Ar, float* out, float* m, float* d, void* workspace,
                       size_t workspace_bytes, void* stream);

/* Partitioned fused backward (fast mode) of one rank:
 *   records of the owned rows; K4f over csc_remote -> the partials of other ranks' sources in
 *   dHt_send / dAl_send (nparts*maxrows rows; this rank's block zero); their reduce-scatter
 *   runs on the communicator's stream while K4f over csc_local writes the own sources' terms;
 *   then dHt = own + received + dA_r (x) a_r, dAl = own + received (num_local rows each) and
 *   dA_r (num_local x h) is complete.  comm == NULL: nothing is received -- dHt / dAl hold the
 *   own-source terms (+ the dA_r LP term) and the caller reduces dHt_send / dAl_send.
 *   Supported where gnncg_gat_fast_supported(heads, f). */
int gnncg_gat_bwd_dist(gnncg_comm_t* comm, const gnncg_part_t* part, int heads, int f, float slope,
                       const float* Ht_all, const float* Al_all, const float* Ar, const float* m, const float* d,
                       const float* out, const float* dOut, const float* a_l, const float* a_r, float* dHt,
                       float* dAl, float* dAr, float* dHt_send, float* dAl_send, void* workspace,
                       size_t workspace_bytes, void* stream);

/* ------------------------------------------------- training-step helpers */
/* params -= lr * grad  (train_step). */
int gnncg_sgd_update(int64_t n, float lr, const float* grad, float* param, void* stream);
/* x[0..n) = value (x 16-byte aligned); e.g. the all-ones seed gradient. */
int gnncg_fill(int64_t n, float value, float* x, void* stream);
/* *out = sum of x[0..n) (loss = sum of exits); fixed-order, bitwise reproducible. */
size_t gnncg_sum_workspace(void);
int gnncg_sum(int64_t n, const float* x, float* out, void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GNNCG_B200_H_ */
