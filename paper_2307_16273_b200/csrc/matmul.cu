// matmul.cu — reduce a stacked matmul to a sumcheck at verifier points.
//
// Y[n] = A[n] B[n] (Eq. exm-matmul-batched).  With w, u1, u3 drawn from the
// transcript (D3a), the restrictions
//     At[k][n] = sum_a beta(u1, a) A[n][a][k]        Bt[k][n] = sum_c B[n][k][c] beta(u3, c)
// turn the claim Y~(w, u1, u3) = sum_{k,n} beta(w, n) At[k][n] Bt[k][n] into the product sumcheck of
// sumcheck.cu (m = logN + logD2, n_eq = logN, K = 2).  Each restriction reads the int32 operand once
// with lazy 320-bit int32 x Fr accumulation (tables.cuh): column sums when the summed index is the
// row index of the stored operand, warp row-dots when it is the column index.
#include "matmul.cuh"
#include "tables.cuh"

namespace zk {

// claim = sum_i beta(w, i mod N) At[i] Bt[i]
__global__ void __launch_bounds__(256) k_mm_claim(const fr_t* At, const fr_t* Bt, const fr_t* Ew, uint64_t total,
                                                  uint64_t nmask, fr_t* partials, unsigned int* ticket, fr_t* out) {
    fr_t acc[1] = {fr_zero()};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x)
        acc[0] = fr_add(acc[0], fr_mul(fr_mul(fr_load(&At[i]), fr_load(&Bt[i])), fr_load(&Ew[i & nmask])));
    fr_t tot[1];
    if (grid_reduce_fr<1>(acc, partials, ticket, tot)) fr_store(out, tot[0]);
}

void matmul_reduce_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* A, const int32_t* B, const zk_mm_shape& sh,
                       fr_t* At, fr_t* Bt, fr_t* d_pts /* logN+logD1+logD3, Montgomery */,
                       uint8_t* d_pts_canon, fr_t* d_claim, Scratch& s) {
    const uint32_t lN = sh.logN, l1 = sh.logD1, l2 = sh.logD2, l3 = sh.logD3;
    ZK_REQUIRE(lN <= 20 && l1 <= 12 && l2 <= 20 && l3 <= 12 && lN + l2 <= 34, ZK_ERR_ARG,
               "matmul: unsupported shape (D1, D3 <= 4096)");
    const uint64_t N = 1ull << lN, D1 = 1ull << l1, D2 = 1ull << l2, D3 = 1ull << l3;
    uint8_t hdr[16];
    const uint32_t hv[4] = {lN, l1, l2, l3};
    for (int i = 0; i < 4; i++)
        for (int k = 0; k < 4; k++) hdr[4 * i + k] = (uint8_t)(hv[i] >> (8 * k));
    tr_absorb_host(tr, "mm/hdr", hdr, 16);
    fr_t* w = d_pts;
    fr_t* u1 = d_pts + lN;
    fr_t* u3 = d_pts + lN + l1;
    {   // one launch for the three vectors (the same chain as three draws)
        const char* tags[3] = {"mm/w", "mm/u1", "mm/u3"};
        const uint32_t ns[3] = {lN, l1, l3};
        fr_t* outs[3] = {w, u1, u3};
        uint8_t* canon[3] = {d_pts_canon, d_pts_canon ? d_pts_canon + 32ull * lN : nullptr,
                             d_pts_canon ? d_pts_canon + 32ull * (lN + l1) : nullptr};
        tr_challenges_multi_dev(tr, 3, tags, ns, outs, canon);
    }
    fr_t* E1 = s.alloc<fr_t>(D1);
    fr_t* E3 = s.alloc<fr_t>(D3);
    eq_table_r2_dev(ctx, u1, l1, E1, s);
    eq_table_r2_dev(ctx, u3, l3, E3, s);
    // At[k][n]
    if (!sh.trans_a) {   // A stored [N][D1][D2]: column sums over a
        colsum_i32(ctx, A, N, (uint32_t)D1, (uint32_t)D2, E1, At, s);
    } else if (rowdot_tc_ok(N * D2, (uint32_t)D1)) {   // A stored [N][D2][D1]: row dots on the tensor cores
        rowdot_tc(ctx, A, N * D2, (uint32_t)D1, E1, At, D2, l2, N, s);
    } else {             // one warp per (n, k) row
        ZK_LAUNCH(ctx, k_rowdot_i32<LoadPlain>, grid_for(ctx, N * D2 * 32, 256, 8), 256, 0, LoadPlain{A}, N * D2,
                  (uint32_t)D1, E1, At, D2, l2, N);
    }
    // Bt[k][n]
    if (!sh.trans_b && rowdot_tc_ok(N * D2, (uint32_t)D3)) {   // B stored [N][D2][D3]: row dots over c, tensor cores
        rowdot_tc(ctx, B, N * D2, (uint32_t)D3, E3, Bt, D2, l2, N, s);
    } else if (!sh.trans_b) {
        ZK_LAUNCH(ctx, k_rowdot_i32<LoadPlain>, grid_for(ctx, N * D2 * 32, 256, 8), 256, 0, LoadPlain{B}, N * D2,
                  (uint32_t)D3, E3, Bt, D2, l2, N);
    } else {             // B stored [N][D3][D2]: column sums over c
        colsum_i32(ctx, B, N, (uint32_t)D3, (uint32_t)D2, E3, Bt, s);
    }
    // claim
    fr_t* Ew = s.alloc<fr_t>(N);
    eq_table_dev(ctx, w, lN, nullptr, Ew, s);
    unsigned int g = grid_for(ctx, N * D2, 256, 2);
    fr_t* part = s.alloc<fr_t>(g);
    unsigned int* ticket = s.alloc_zero<unsigned int>(1);
    ZK_LAUNCH(ctx, k_mm_claim, g, 256, 0, At, Bt, Ew, N * D2, N - 1, part, ticket, d_claim);
}

}  // namespace zk
