// matmul.cuh — restriction of a stacked matmul to sumcheck tables (row a3).
#pragma once
#include "common.cuh"

namespace zk {
void matmul_reduce_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* A, const int32_t* B, const zk_mm_shape& sh,
                       fr_t* At, fr_t* Bt, fr_t* d_pts, uint8_t* d_pts_canon, fr_t* d_claim, Scratch& s);
}
