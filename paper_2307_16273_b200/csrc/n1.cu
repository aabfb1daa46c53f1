// n1.cu — SURVEY §8(f) N1: the re-indexing sumcheck (Eq. sc-reindex, D20)
// and the zkReLU aux-claim merge (D21).  Both reduce several claims to one
// with a short product sumcheck (rows a4-a6 engine) over tables built here:
//  * re-indexing: C(i) = sum_k r_k sum_j beta(u_k, j) [map_k[j] == i]  (scatter of scaled eq tables) and
//    X_u(i) = X~(u, i) = sum_d beta(u, d) X[i][d]  (one warp per slice, lazy int32 x Fr accumulation);
//  * merge: T(s, j) = sum_i beta(v, i) bit_j(word_s[i])  (one warp per chunk of entries, lane j owns bit
//    j: lazy additions of the eq weight, no product per entry beyond the eq table itself) and the
//    32-entry weight table W(s, j).
#include <cstring>
#include <vector>

#include "sumcheck.cuh"
#include "tables.cuh"

using namespace zk;

namespace zk {

// C[map[j]] += E[j] for one view (map injective, checked on the host; 0xffffffff = empty slot)
__global__ void k_scatter_add(const uint32_t* map, uint64_t n, const fr_t* E, fr_t* C) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = map[j];
        if (i == 0xffffffffu) continue;
        fr_store(&C[i], fr_add(fr_load_l2(&C[i]), fr_load(&E[j])));
    }
}

// out = sum_k a[k] b[k] (K small; one thread)
__global__ void k_lincomb(const fr_t* a, const fr_t* b, uint32_t K, fr_t* out) {
    fr_t acc = fr_zero();
    for (uint32_t k = 0; k < K; k++) acc = fr_add(acc, fr_mul_cold(fr_load(&a[k]), fr_load(&b[k])));
    fr_store(out, acc);
}

// merge: claim = f0 + rho f1 + rho^2 f2;  W(s, j) for s in {0, 1}, j < B (flat s * B + j):
// [s = 0] (beta(w, j) + rho^2 [j = QR - 1]) + [s = 1] rho beta(w, j)
__global__ void k_merge_setup(const fr_t* f, const fr_t* rho_p, const fr_t* Ew, uint32_t B, uint32_t QR, fr_t* claim,
                              fr_t* W) {
    const fr_t rho = fr_load(rho_p);
    const fr_t rho2 = fr_mul_cold(rho, rho);
    const uint32_t t = threadIdx.x;
    if (t == 0)
        fr_store(claim, fr_add(fr_add(fr_load(&f[0]), fr_mul_cold(rho, fr_load(&f[1]))), fr_mul_cold(rho2, fr_load(&f[2]))));
    if (t < 2 * B) {
        const uint32_t s = t / B, j = t % B;
        const fr_t e = fr_load(&Ew[j]);
        fr_t w = s ? fr_mul_cold(rho, e) : e;
        if (!s && j == QR - 1) w = fr_add(w, rho2);
        fr_store(&W[t], w);
    }
}

// lazy 9-limb accumulation of Fr values (no reduction until the end; < 2^32 additions)
__device__ __forceinline__ void lazy_add9(uint32_t (&a)[9], const fr_t& e) {
    asm("add.cc.u32  %0, %0, %9;\n\t"
        "addc.cc.u32 %1, %1, %10;\n\t"
        "addc.cc.u32 %2, %2, %11;\n\t"
        "addc.cc.u32 %3, %3, %12;\n\t"
        "addc.cc.u32 %4, %4, %13;\n\t"
        "addc.cc.u32 %5, %5, %14;\n\t"
        "addc.cc.u32 %6, %6, %15;\n\t"
        "addc.cc.u32 %7, %7, %16;\n\t"
        "addc.u32    %8, %8, 0;"
        : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]), "+r"(a[8])
        : "r"(e.v[0]), "r"(e.v[1]), "r"(e.v[2]), "r"(e.v[3]), "r"(e.v[4]), "r"(e.v[5]), "r"(e.v[6]), "r"(e.v[7]));
}
// sum (as an integer < 2^288) -> Fr: REDC(sum) * R^2 via Montgomery = sum mod p (Montgomery form kept)
__device__ __forceinline__ fr_t lazy_finish9(const uint32_t (&a)[9]) {
    const uint32_t w[10] = {a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8], 0};
    return fr_mul(fr_redc_wide(w), ZK_R2);
}

// T(s, j) partial sums without a 2^logD eq table: beta(v, i) = LO[i mod 2^lo] * HI[i >> lo], one block
// per HI value h.  Each warp stages 32 entries (LO weight, both words) in shared memory, then lane j
// walks them (broadcast reads) and adds the LO weight lazily (9-limb, no reduction) when bit j is set;
// the lazy sums are closed once per warp, added over the block and multiplied by HI[h] once.
__global__ void __launch_bounds__(256) k_aux_colsum(const int32_t* Z, const int32_t* GA, const fr_t* LO,
                                                    const fr_t* HI, uint32_t lo, uint32_t qr_mask, fr_t* partials) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __shared__ fr_t se[8][32];
    __shared__ uint2 sw[8][32];
    uint32_t az[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, ag[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    const uint64_t base = (uint64_t)blockIdx.x << lo, n = 1ull << lo;
    for (uint64_t c = (uint64_t)wid * 32; c < n; c += (uint64_t)nw * 32) {
        const uint64_t x = c + lane;
        if (x < n) {
            se[wid][lane] = fr_load(&LO[x]);
            sw[wid][lane] = make_uint2((uint32_t)__ldg(Z + base + x) & qr_mask, (uint32_t)__ldg(GA + base + x) & qr_mask);
        } else {
            se[wid][lane] = fr_zero();
            sw[wid][lane] = make_uint2(0u, 0u);
        }
        __syncwarp();
#pragma unroll 4
        for (int k = 0; k < 32; k++) {
            const uint2 w = sw[wid][k];
            if (((w.x | w.y) >> lane) & 1) {
                const fr_t e = se[wid][k];
                if ((w.x >> lane) & 1) lazy_add9(az, e);
                if ((w.y >> lane) & 1) lazy_add9(ag, e);
            }
        }
        __syncwarp();
    }
    __shared__ fr_t sm[8][64];
    sm[wid][lane] = lazy_finish9(az);
    sm[wid][32 + lane] = lazy_finish9(ag);
    __syncthreads();
    if (threadIdx.x < 64) {
        fr_t acc = sm[0][threadIdx.x];
        for (int w = 1; w < nw; w++) acc = fr_add(acc, sm[w][threadIdx.x]);
        fr_store(&partials[blockIdx.x * 64ull + threadIdx.x], fr_mul(acc, fr_load(&HI[blockIdx.x])));
    }
}

// T[s * B + j] = sum over blocks (j < 32; zero for 32 <= j < B): 4 warps per output cell
__global__ void k_aux_colsum_reduce(const fr_t* partials, uint32_t nblocks, uint32_t B, fr_t* T) {
    const uint32_t cell = blockIdx.x, s = cell / B, j = cell % B;
    __shared__ fr_t sm[4];
    fr_t acc = fr_zero();
    if (j < 32)
        for (uint32_t b = threadIdx.x; b < nblocks; b += blockDim.x) acc = fr_add(acc, fr_load(&partials[b * 64ull + s * 32 + j]));
    for (int off = 16; off > 0; off >>= 1) acc = fr_add(acc, fr_shfl_down(acc, off));
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (uint32_t w = 1; w < blockDim.x / 32; w++) acc = fr_add(acc, sm[w]);
        fr_store(&T[cell], acc);
    }
}

// canonical 32-byte encodings (already checked < p by the producer) -> Montgomery
__global__ void k_canon_to_mont(const uint8_t* in, uint32_t n, fr_t* out) {
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        fr_t x;
        for (int l = 0; l < 8; l++)
            x.v[l] = (uint32_t)in[32 * i + 4 * l] | ((uint32_t)in[32 * i + 4 * l + 1] << 8) |
                     ((uint32_t)in[32 * i + 4 * l + 2] << 16) | ((uint32_t)in[32 * i + 4 * l + 3] << 24);
        fr_store(&out[i], fr_from_canonical(x));
    }
}

// The merge (D21) from device-resident point and finals (Montgomery); proof and point to device memory.
static void relu_merge_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_Z, const int32_t* d_GA, uint32_t logD,
                           uint32_t Q, uint32_t R, const fr_t* pt, const fr_t* f, uint8_t* d_proof, uint8_t* d_point,
                           Scratch& s) {
    const uint32_t QR = Q + R;
    uint32_t logB = 0;
    while ((1u << logB) < QR) logB++;
    const uint32_t B = 1u << logB, m = logB + 1;
    const uint64_t D = 1ull << logD;
    fr_t* rho = s.alloc<fr_t>(1);
    tr_challenges_dev(tr, "relu/merge", 1, rho, nullptr);
    ScStatement S;
    memset(&S, 0, sizeof S);
    S.m = m;
    S.n_eq = 0;
    S.K = 2;
    S.d_claim = s.alloc<fr_t>(1);
    S.claim_given = true;
    // beta(v, i) = LO[i mod 2^lo] HI[i >> lo]: 2^lo entries per block of k_aux_colsum
    const uint32_t lo = logD < 12 ? logD : 12, hi = logD - lo;
    fr_t* Ew = s.alloc<fr_t>(B);
    fr_t* LO = s.alloc<fr_t>(1ull << lo);
    fr_t* HI = s.alloc<fr_t>(1ull << hi);
    EqJob jobs[3] = {EqJob{pt, logB, nullptr, 0, Ew}, EqJob{pt + logB, lo, nullptr, 0, LO},
                     EqJob{pt + logB + lo, hi, nullptr, 0, HI}};
    eq_tables_batch(ctx, 3, jobs, s);
    fr_t* W = s.alloc<fr_t>(2 * B);
    ZK_LAUNCH(ctx, k_merge_setup, 1, 64, 0, f, (const fr_t*)rho, (const fr_t*)Ew, B, QR, S.d_claim, W);
    // T(s, j) = sum_i beta(v, i) bit_j(word_s[i])
    const unsigned int grid = 1u << hi;
    fr_t* part = s.alloc<fr_t>((size_t)grid * 64);
    const uint32_t qr_mask = QR >= 32 ? 0xffffffffu : ((1u << QR) - 1);
    ZK_LAUNCH(ctx, k_aux_colsum, grid, 256, 0, d_Z, d_GA, (const fr_t*)LO, (const fr_t*)HI, lo, qr_mask, part);
    fr_t* T = s.alloc<fr_t>(2 * B);
    ZK_LAUNCH(ctx, k_aux_colsum_reduce, 2 * B, 128, 0, (const fr_t*)part, grid, B, T);
    (void)D;
    S.tables[0] = T;
    S.tables[1] = W;
    S.d_proof = d_proof;
    S.d_r = s.alloc<fr_t>(m);
    S.d_point = d_point;
    sumcheck_prove_dev(ctx, tr, S, s);
}

static void copy_proof_out(zk_ctx* ctx, const ScStatement& S, uint32_t m, uint8_t* proof, zk_fr* point_out,
                           zk_fr* finals_out) {
    const uint64_t plen = sumcheck_proof_len(m, 2);
    if (proof) ZK_CUDA(cudaMemcpyAsync(proof, S.d_proof, plen, cudaMemcpyDeviceToHost, ctx->stream));
    if (point_out) ZK_CUDA(cudaMemcpyAsync(point_out, S.d_point, 32ull * m, cudaMemcpyDeviceToHost, ctx->stream));
    if (finals_out)
        ZK_CUDA(cudaMemcpyAsync(finals_out, S.d_proof + 44 + 32ull * m * 3, 64, cudaMemcpyDeviceToHost, ctx->stream));
    ZK_CUDA(cudaStreamSynchronize(ctx->stream));
}

static bool proof_len_check(uint64_t plen, uint8_t* proof, uint64_t* proof_len) {   // true: size query only
    if (!proof_len) return false;
    const bool query = !proof;
    if (proof && *proof_len < plen) {
        *proof_len = plen;
        throw ZkError{ZK_ERR_ARG, "proof buffer too small"};
    }
    *proof_len = plen;
    return query;
}

}  // namespace zk

#define N1_BEGIN(ctx)                                                                                  \
    if (!(ctx)) return ZK_ERR_ARG;                                                                     \
    try {                                                                                              \
        ZK_CUDA(cudaSetDevice((ctx)->device));
#define N1_END(ctx)                                                                                    \
    }                                                                                                  \
    catch (const ::zk::ZkError& e) {                                                                   \
        (ctx)->err = e.msg;                                                                            \
        return e.st;                                                                                   \
    }                                                                                                  \
    catch (const std::exception& e) {                                                                  \
        (ctx)->err = e.what();                                                                         \
        return ZK_ERR_INTERNAL;                                                                        \
    }                                                                                                  \
    return ZK_OK;

extern "C" {

zk_status zk_reindex_prove(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_X, uint32_t n, uint32_t d, uint32_t K,
                           const zk_view* views, const zk_fr* u, const zk_fr* claims, uint8_t* proof,
                           uint64_t* proof_len, zk_fr* point_out, zk_fr* finals_out) {
    N1_BEGIN(ctx)
    ZK_REQUIRE(tr && d_X && views && claims && (u || !d), ZK_ERR_ARG, "null argument");
    ZK_REQUIRE(n >= 1 && n <= 30 && d <= 34 && n + d <= 40 && K >= 1 && K <= 32, ZK_ERR_ARG, "bad re-indexing shape");
    if (proof_len_check(sumcheck_proof_len(n, 2), proof, proof_len)) return ZK_OK;
    const uint64_t N = 1ull << n;
    // host-side checks: every map injective into [0, N) (empty slots excepted)
    std::vector<uint8_t> seen(N);
    for (uint32_t k = 0; k < K; k++) {
        ZK_REQUIRE(views[k].logN <= 30 && (views[k].map || !views[k].logN) && (views[k].u || !views[k].logN), ZK_ERR_ARG,
                   "bad view");
        std::fill(seen.begin(), seen.end(), 0);
        for (uint64_t j = 0; j < (1ull << views[k].logN); j++) {
            const uint32_t i = views[k].map ? views[k].map[j] : 0u;
            if (i == 0xffffffffu) continue;
            ZK_REQUIRE(i < N, ZK_ERR_RANGE, "view slot outside the stack");
            ZK_REQUIRE(!seen[i], ZK_ERR_ARG, "view map not injective");
            seen[i] = 1;
        }
    }
    Scratch s(ctx);
    // transcript (D20): "rx/hdr" (n, d, K, n_k...) | "rx/claims" | r_k = "rx/r" x K
    std::vector<uint32_t> hdr = {n, d, K};
    for (uint32_t k = 0; k < K; k++) hdr.push_back(views[k].logN);
    std::vector<uint8_t> hb(4 * hdr.size());
    for (size_t i = 0; i < hdr.size(); i++)
        for (int b = 0; b < 4; b++) hb[4 * i + b] = (uint8_t)(hdr[i] >> (8 * b));
    tr_absorb_host(tr, "rx/hdr", hb.data(), hb.size());
    fr_t* cl = s.alloc<fr_t>(K);
    upload_points(ctx, claims, K, cl, s);
    ZK_LAUNCH(ctx, k_tr_absorb_frs, 1, 32, 0, tr->d_st, make_tag("rx/claims"), (const fr_t*)cl, K, (uint8_t*)nullptr);
    fr_t* rk = s.alloc<fr_t>(K);
    tr_challenges_dev(tr, "rx/r", K, rk, nullptr);
    ScStatement S;
    memset(&S, 0, sizeof S);
    S.m = n;
    S.n_eq = 0;
    S.K = 2;
    S.d_claim = s.alloc<fr_t>(1);
    S.claim_given = true;
    ZK_LAUNCH(ctx, k_lincomb, 1, 1, 0, (const fr_t*)rk, (const fr_t*)cl, K, S.d_claim);
    // C(i) = sum_k r_k sum_j beta(u_k, j) [map_k[j] == i]
    fr_t* C = s.alloc_zero<fr_t>(N);
    for (uint32_t k = 0; k < K; k++) {
        const uint64_t nk = 1ull << views[k].logN;
        fr_t* uk = s.alloc<fr_t>(views[k].logN ? views[k].logN : 1);
        if (views[k].logN) upload_points(ctx, views[k].u, views[k].logN, uk, s);
        fr_t* E = s.alloc<fr_t>(nk);
        eq_table_dev(ctx, uk, views[k].logN, rk + k, E, s);
        uint32_t* dmap = s.alloc<uint32_t>(nk);
        if (views[k].map) {
            ZK_CUDA(cudaMemcpyAsync(dmap, views[k].map, nk * 4, cudaMemcpyHostToDevice, ctx->stream));
        } else {
            ZK_CUDA(cudaMemsetAsync(dmap, 0, 4, ctx->stream));
        }
        ZK_LAUNCH(ctx, k_scatter_add, grid_for(ctx, nk, 256, 4), 256, 0, (const uint32_t*)dmap, nk, (const fr_t*)E, C);
    }
    // X_u(i) = sum_c beta(u, c) X[i][c]
    fr_t* Xu = s.alloc<fr_t>(N);
    fr_t* du = s.alloc<fr_t>(d ? d : 1);
    if (d) upload_points(ctx, u, d, du, s);
    fr_t* E2 = s.alloc<fr_t>(1ull << d);
    eq_table_r2_dev(ctx, du, d, E2, s);
    ZK_LAUNCH(ctx, k_rowdot_i32<LoadPlain>, grid_for(ctx, N * 32, 256, 8), 256, 0, LoadPlain{d_X}, N, 1u << d,
              (const fr_t*)E2, Xu, N, n, (uint64_t)1);
    S.tables[0] = C;
    S.tables[1] = Xu;
    S.d_proof = s.alloc<uint8_t>(sumcheck_proof_len(n, 2));
    S.d_r = s.alloc<fr_t>(n);
    S.d_point = s.alloc<uint8_t>(32ull * n);
    sumcheck_prove_dev(ctx, tr, S, s);
    copy_proof_out(ctx, S, n, proof, point_out, finals_out);
    N1_END(ctx)
}

zk_status zk_relu_merge(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_Z, const int32_t* d_GA, uint32_t logD,
                        uint32_t Q, uint32_t R, const zk_fr* point, const zk_fr* finals, uint8_t* proof,
                        uint64_t* proof_len, zk_fr* point_out, zk_fr* merged_out) {
    N1_BEGIN(ctx)
    ZK_REQUIRE(tr && d_Z && d_GA && point && finals, ZK_ERR_ARG, "null argument");
    const uint32_t QR = Q + R;
    ZK_REQUIRE(Q >= 1 && R >= 1 && Q <= 32 && R <= 32 && QR <= 32 && logD >= 1 && logD <= 32, ZK_ERR_ARG, "bad zkReLU shape");
    uint32_t logB = 0;
    while ((1u << logB) < QR) logB++;
    const uint32_t m = logB + 1;
    if (proof_len_check(sumcheck_proof_len(m, 2), proof, proof_len)) return ZK_OK;
    Scratch s(ctx);
    fr_t* pt = s.alloc<fr_t>(logB + logD);
    upload_points(ctx, point, logB + logD, pt, s);
    fr_t* f = s.alloc<fr_t>(3);
    upload_points(ctx, finals, 3, f, s);
    ScStatement S;
    memset(&S, 0, sizeof S);
    S.d_proof = s.alloc<uint8_t>(sumcheck_proof_len(m, 2));
    S.d_point = s.alloc<uint8_t>(32ull * m);
    relu_merge_dev(ctx, tr, d_Z, d_GA, logD, Q, R, pt, f, S.d_proof, S.d_point, s);
    copy_proof_out(ctx, S, m, proof, point_out, merged_out);
    N1_END(ctx)
}

zk_status zk_relu_merge_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_Z, const int32_t* d_GA, uint32_t logD,
                            uint32_t Q, uint32_t R, const uint8_t* d_relu_out, uint8_t* d_out, uint64_t* out_len) {
    N1_BEGIN(ctx)
    ZK_REQUIRE(tr && d_Z && d_GA && d_relu_out, ZK_ERR_ARG, "null argument");
    const uint32_t QR = Q + R;
    ZK_REQUIRE(Q >= 1 && R >= 1 && Q <= 32 && R <= 32 && QR <= 32 && logD >= 1 && logD <= 30, ZK_ERR_ARG, "bad zkReLU shape");
    uint32_t logB = 0;
    while ((1u << logB) < QR) logB++;
    const uint32_t m = logB + 1;
    const uint64_t plen = sumcheck_proof_len(m, 2), off_pt = (plen + 15) & ~15ull;
    if (out_len) {
        const bool query = !d_out;
        if (d_out && *out_len < off_pt + 32ull * m) {
            *out_len = off_pt + 32ull * m;
            throw ZkError{ZK_ERR_ARG, "output buffer too small"};
        }
        *out_len = off_pt + 32ull * m;
        if (query) return ZK_OK;
    }
    ZK_REQUIRE(d_out && ((uintptr_t)d_out & 15) == 0, ZK_ERR_ARG, "d_out must be 16-byte aligned");
    // the zkReLU output (zk_relu_prove_dev layout): proof | pad | point; its finals end the proof
    const uint64_t rplen = 12 + 128 + 128ull * (logB + logD) + 96, roff = (rplen + 15) & ~15ull;
    Scratch s(ctx);
    fr_t* pt = s.alloc<fr_t>(logB + logD);
    fr_t* f = s.alloc<fr_t>(3);
    ZK_LAUNCH(ctx, k_canon_to_mont, 1, 64, 0, d_relu_out + roff, logB + logD, pt);
    ZK_LAUNCH(ctx, k_canon_to_mont, 1, 64, 0, d_relu_out + rplen - 96, 3u, f);
    relu_merge_dev(ctx, tr, d_Z, d_GA, logD, Q, R, pt, f, d_out, d_out + off_pt, s);
    N1_END(ctx)
}

}  // extern "C"
