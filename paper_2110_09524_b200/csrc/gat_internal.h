// SPDX-License-Identifier: Apache-2.0
// Internal hooks between gat.cu and dist.cu (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>

#include "gnncg_b200.h"

namespace gnncg_b200 {

// flags of gat_bwd_src_fused_impl (gat.cu)
constexpr int kFusedKeepDar = 1;  // do not zero dA_r: accumulate into the caller's values
constexpr int kFusedNoLpDar = 2;  // leave the dA_r (x) a_r LP term of dHt to the caller

// One fp32 K4f pass over `csc_src` (rows = sources, neighbours = local destination rows
// [0, num_local)): dHt / dAl rows of the index written (with the dA_l (x) a_l LP term),
// dA_r += dz by global reductions (zeroed first when zero_dar).  No dA_r (x) a_r term.
int gat_bwd_src_fused_pass(const gnncg_index_t* csc_src, const gnncg_sched_t* sched, int h, int f, float slope,
                           int64_t num_local, const float* Ht, const float* Al, const float* dst_rec,
                           const float* dOut, const float* a_l, const float* a_r, float* dHt, float* dAl, float* dAr,
                           bool zero_dar, void* ws, size_t ws_bytes, cudaStream_t stream);

// dHt[r, :] += dA_r[r] (x) a_r for r in [0, rows).
int gat_lp_dar(int64_t rows, int h, int f, const float* dAr, const float* a_r, float* dHt, cudaStream_t s);

}  // namespace gnncg_b200
