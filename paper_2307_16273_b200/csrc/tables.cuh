// tables.cuh — int32 x Fr lazy accumulation and generic reduction kernels shared by
// the MLE evaluator (row a2), the matmul restriction (row a3) and the zkReLU claims (row a8).
//
// Lazy accumulation: a weight table E' holding eq * R (i.e. stored as eq * R^2 mod p, "double
// Montgomery") is multiplied by u = v + 2^31 (the int32 value biased to u32) and summed as a plain
// 320-bit integer, 16 IMAD per element, with ONE Montgomery reduction at the end:
//   REDC(sum u E') = sum (v + 2^31) eq R = mont(sum v eq) + mont(2^31) * sum eq,
// and sum eq = 1 over a full eq table, so the bias is removed by subtracting mont(2^31).
// Bound: <= 2^16 terms of < 2^32 * 2^255 stay below 2^303 < 10 limbs, far below p * 2^256.
#pragma once
#include "common.cuh"

namespace zk {

// acc[0..9] += e[0..7] * u
#define ZK_MAC_WIDE(acc, e, u)                                                                         \
    asm("mad.lo.cc.u32  %0, %10, %18, %0;\n\t"                                                         \
        "madc.lo.cc.u32 %1, %11, %18, %1;\n\t"                                                         \
        "madc.lo.cc.u32 %2, %12, %18, %2;\n\t"                                                         \
        "madc.lo.cc.u32 %3, %13, %18, %3;\n\t"                                                         \
        "madc.lo.cc.u32 %4, %14, %18, %4;\n\t"                                                         \
        "madc.lo.cc.u32 %5, %15, %18, %5;\n\t"                                                         \
        "madc.lo.cc.u32 %6, %16, %18, %6;\n\t"                                                         \
        "madc.lo.cc.u32 %7, %17, %18, %7;\n\t"                                                         \
        "addc.cc.u32    %8, %8, 0;\n\t"                                                                \
        "addc.u32       %9, %9, 0;\n\t"                                                                \
        "mad.hi.cc.u32  %1, %10, %18, %1;\n\t"                                                         \
        "madc.hi.cc.u32 %2, %11, %18, %2;\n\t"                                                         \
        "madc.hi.cc.u32 %3, %12, %18, %3;\n\t"                                                         \
        "madc.hi.cc.u32 %4, %13, %18, %4;\n\t"                                                         \
        "madc.hi.cc.u32 %5, %14, %18, %5;\n\t"                                                         \
        "madc.hi.cc.u32 %6, %15, %18, %6;\n\t"                                                         \
        "madc.hi.cc.u32 %7, %16, %18, %7;\n\t"                                                         \
        "madc.hi.cc.u32 %8, %17, %18, %8;\n\t"                                                         \
        "addc.u32       %9, %9, 0;"                                                                    \
        : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3]), "+r"(acc[4]), "+r"(acc[5]),          \
          "+r"(acc[6]), "+r"(acc[7]), "+r"(acc[8]), "+r"(acc[9])                                       \
        : "r"(e.v[0]), "r"(e.v[1]), "r"(e.v[2]), "r"(e.v[3]), "r"(e.v[4]), "r"(e.v[5]), "r"(e.v[6]),  \
          "r"(e.v[7]), "r"(u))

// acc[0..9] += b[0..9]
__device__ __forceinline__ void wide_add10(uint32_t (&a)[10], const uint32_t (&b)[10]) {
    asm("add.cc.u32  %0, %0, %10;\n\t"
        "addc.cc.u32 %1, %1, %11;\n\t"
        "addc.cc.u32 %2, %2, %12;\n\t"
        "addc.cc.u32 %3, %3, %13;\n\t"
        "addc.cc.u32 %4, %4, %14;\n\t"
        "addc.cc.u32 %5, %5, %15;\n\t"
        "addc.cc.u32 %6, %6, %16;\n\t"
        "addc.cc.u32 %7, %7, %17;\n\t"
        "addc.cc.u32 %8, %8, %18;\n\t"
        "addc.u32    %9, %9, %19;"
        : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
          "+r"(a[8]), "+r"(a[9])
        : "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(b[4]), "r"(b[5]), "r"(b[6]), "r"(b[7]), "r"(b[8]),
          "r"(b[9]));
}

__device__ __forceinline__ void wide_warp_reduce(uint32_t (&a)[10]) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        uint32_t o[10];
#pragma unroll
        for (int i = 0; i < 10; i++) o[i] = __shfl_down_sync(0xffffffffu, a[i], off);
        wide_add10(a, o);
    }
}

// Final value of a lazy accumulator: Montgomery form of sum v * eq.
__device__ __forceinline__ fr_t wide_finish(const uint32_t (&a)[10]) {
    return fr_sub(fr_redc_wide(a), ZK_TWO31_MONT);
}

// ---------------------------------------------------------------- element loaders (int32 views)
struct LoadPlain {
    const int32_t* p;
    __device__ __forceinline__ int32_t operator()(uint64_t i) const { return __ldg(p + i); }
};
// A = 1{Z >= 0} round(Z / 2^R) (Lemma 1; half-up D9)
struct LoadReluA {
    const int32_t* z;
    uint32_t R;
    __device__ __forceinline__ int32_t operator()(uint64_t i) const {
        int64_t v = __ldg(z + i);
        return v >= 0 ? (int32_t)((v + (1ll << (R - 1))) >> R) : 0;
    }
};
// G_Z = 1{Z >= 0} round(G_A / 2^R) (Lemma 1)
struct LoadReluGZ {
    const int32_t* z;
    const int32_t* g;
    uint32_t R;
    __device__ __forceinline__ int32_t operator()(uint64_t i) const {
        int64_t zv = __ldg(z + i), gv = __ldg(g + i);
        return zv >= 0 ? (int32_t)((gv + (1ll << (R - 1))) >> R) : 0;
    }
};

// Z' = round(Z / 2^R) (half-up D9), the rescale of the top layer (D26)
struct LoadRound {
    const int32_t* z;
    uint32_t R;
    __device__ __forceinline__ int32_t operator()(uint64_t i) const {
        const int64_t v = __ldg(z + i);
        return (int32_t)((v + (1ll << (R - 1))) >> R);
    }
};
// aux(i, j) = bit j of Z[i] (zero for j >= QR), flat index i * 2^logB + j (the rescale's aux bits, D26)
struct LoadBits {
    const int32_t* z;
    uint32_t logB, QR;
    __device__ __forceinline__ int32_t operator()(uint64_t x) const {
        const uint32_t j = (uint32_t)(x & ((1ull << logB) - 1));
        return j < QR ? (int32_t)(((uint32_t)__ldg(z + (x >> logB)) >> j) & 1u) : 0;
    }
};

// One warp per row r of an int32 matrix viewed through `load` (row-major, `cols` entries per row,
// rows < nrows): out[map(r)] = sum_c M[r][c] * eq[c], with E2 = eq table scaled by R (double Montgomery).
// map(r) = (r & (inner - 1)) * outer + (r >> log_inner)   (restriction layout [k][n]); inner = nrows gives identity.
// (Measured: unrolling eight loads per lane, or four rows per warp sharing the eq loads, were slower.)
template <class Load>
__global__ void __launch_bounds__(256) k_rowdot_i32(Load load, uint64_t nrows, uint32_t cols, const fr_t* E2,
                                                    fr_t* out, uint64_t inner, uint32_t log_inner, uint64_t outer) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = warp; r < nrows; r += nwarps) {
        uint32_t acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        const uint64_t base = r * cols;
        for (uint32_t c = lane; c < cols; c += 32) {
            uint32_t u = (uint32_t)load(base + c) + 0x80000000u;
            fr_t e = fr_load(&E2[c]);
            ZK_MAC_WIDE(acc, e, u);
        }
        wide_warp_reduce(acc);
        if (lane == 0) {
            uint64_t o = (r & (inner - 1)) * outer + (r >> log_inner);
            fr_store(&out[o], wide_finish(acc));
        }
    }
}

// Work item (s, n, c) of M[N][rows][cols] (c fastest): the lazy sum over rows [s rows/S, (s+1) rows/S) of
// eq[r] * M[n][r][c] (E2 double Montgomery).  S = 1: out[c * N + n] directly; S > 1: the 10-limb partial
// to partials[item] (exact integers, summed by k_colsum_finish).  Sixteen loads in flight per thread and
// two lazy accumulators (even / odd rows), so consecutive MACs are independent carry chains.
template <class Load>
__global__ void __launch_bounds__(128) k_colsum_i32(Load load, uint64_t N, uint32_t rows, uint32_t cols, const fr_t* E2,
                                                    fr_t* out, uint32_t S, uint32_t* partials) {
    const uint64_t outputs = N * cols, total = outputs * S;
    const uint32_t chunk = rows / S;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t o = t % outputs, n = o / cols, c = o % cols;
        const uint32_t sp = (uint32_t)(t / outputs), r0 = sp * chunk, r1 = r0 + chunk;
        uint32_t acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        uint32_t acc2[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        const uint64_t base = n * (uint64_t)rows * cols + c;
        uint32_t r = r0;
        for (; r + 15 < r1; r += 16) {
            uint32_t u[16];
#pragma unroll
            for (int k = 0; k < 16; k++) u[k] = (uint32_t)load(base + (uint64_t)(r + k) * cols) + 0x80000000u;
#pragma unroll
            for (int k = 0; k < 16; k += 2) {
                const fr_t e0 = fr_load(&E2[r + k]), e1 = fr_load(&E2[r + k + 1]);
                ZK_MAC_WIDE(acc, e0, u[k]);
                ZK_MAC_WIDE(acc2, e1, u[k + 1]);
            }
        }
        for (; r < r1; r++) {
            uint32_t u = (uint32_t)load(base + (uint64_t)r * cols) + 0x80000000u;
            fr_t e = fr_load(&E2[r]);
            ZK_MAC_WIDE(acc, e, u);
        }
        wide_add10(acc, acc2);
        if (S == 1) {
            fr_store(&out[c * N + n], wide_finish(acc));
        } else {
#pragma unroll
            for (int k = 0; k < 10; k++) partials[t * 10 + k] = acc[k];
        }
    }
}
// out[c * N + n] = finish(sum_s partials[(s, n, c)])
__global__ void k_colsum_finish(const uint32_t* partials, uint64_t N, uint32_t cols, uint32_t S, fr_t* out);

// Grid reduction of sum_i a[i] * b[i] (Fr); the last block writes the result to *out.
__global__ void k_dot_fr(const fr_t* a, const fr_t* b, uint64_t n, fr_t* partials, unsigned int* ticket, fr_t* out);

// Host helpers (tables.cu)
// MLE of an int32 table viewed through a loader, at a device point (Montgomery); result to d_out (Montgomery).
void mle_i32_plain(zk_ctx* ctx, const int32_t* d_tab, uint32_t m, const fr_t* d_u, fr_t* d_out, Scratch& s);
// Column sums out[c * N + n] = sum_r E2[r] M[n][r][c] of an int32 stack (k_colsum_i32): one wave of 128-thread
// CTAs, the rows split into S chunks (partials summed by k_colsum_finish) when there are few outputs.
void colsum_i32(zk_ctx* ctx, const int32_t* M, uint64_t N, uint32_t rows, uint32_t cols, const fr_t* E2, fr_t* out,
                Scratch& s);
void mle_i32_relu(zk_ctx* ctx, int kind /*0 A, 1 GZ, 2 Z' = round(Z / 2^R)*/, const int32_t* d_z, const int32_t* d_g, uint32_t R, uint32_t m,
                  const fr_t* d_u, fr_t* d_out, Scratch& s);
// Row dots out[map(r)] = sum_c M[r][c] E2[c] of an int32 matrix on the tensor cores (restrict_tc.cu): same
// results as k_rowdot_i32<LoadPlain>; rowdot_tc_ok says whether the shape is supported (cols % 8 == 0,
// cols <= 4096, >= 1024 rows; ZKDL_ROWDOT_TC=0 disables it).
bool rowdot_tc_ok(uint64_t nrows, uint32_t cols);
// Column sums on the tensor cores (restrict_tc.cu: MN-major int8 MMAs fed by TMA), the same results as
// colsum_i32; colsum_tc_ok: cols % 32 == 0, rows % 32 == 0, 32 <= rows <= 4096, at least one tile per SM
// (ZKDL_COLSUM_TC=0 disables it)
bool colsum_tc_ok(uint64_t N, uint32_t rows, uint32_t cols);
void colsum_tc(zk_ctx* ctx, const int32_t* M, uint64_t N, uint32_t rows, uint32_t cols, const fr_t* E2, fr_t* out,
               Scratch& s);
void rowdot_tc(zk_ctx* ctx, const int32_t* M, uint64_t nrows, uint32_t cols, const fr_t* E2, fr_t* out, uint64_t inner,
               uint32_t log_inner, uint64_t outer, Scratch& s, int use_tma = -1 /* -1: default (ZKDL_ROWDOT_TMA), 0: cp.async producer, 1: TMA */);
void mle_i32_relu4(zk_ctx* ctx, const int32_t* d_z, const int32_t* d_g, uint32_t R, uint32_t m, const fr_t* d_U,
                   fr_t* d_out, Scratch& s);
void mle_fr_dev(zk_ctx* ctx, const fr_t* d_tab, uint32_t m, const fr_t* d_u, fr_t* d_out, Scratch& s);
// eq table scaled by R (for the lazy accumulators)
void eq_table_r2_dev(zk_ctx* ctx, const fr_t* d_u, uint32_t k, fr_t* d_out, Scratch& s);
// Several eq tables in two launches (direct parts, then lo x hi combines): out = scale * beta(u, .)
// over k variables; r2 = 1: scale = R (Montgomery form of R), as eq_table_r2_dev.
constexpr uint32_t EQB_MAX = 16;
struct EqJob {
    const fr_t* u;
    uint32_t k;
    const fr_t* scale;
    int r2;
    fr_t* out;
};
void eq_tables_batch(zk_ctx* ctx, uint32_t n, const EqJob* jobs, Scratch& s);
void embed_i32_dev(zk_ctx* ctx, const int32_t* d_in, uint64_t n, fr_t* d_out);

}  // namespace zk
