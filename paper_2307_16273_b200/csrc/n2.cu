// n2.cu — SURVEY §8(f) N2: Protocol 2's zero form for the aggregated Hadamard product (Eq. tensor-op-aggr
// P:L229-234, Protocol 2 P:L476-502; D22), on the product-sumcheck engine (rows a4-a6)
// with the zero-form round kernel k_sc_zero_round; the loss-gradient family (Eq. fcnn-GZ-last, D24) and the
// top-layer rescale through the bits of Z (D26).
#include <cstring>

#include "sumcheck.cuh"
#include "tables.cuh"

using namespace zk;

namespace zk {

__global__ void k_canon_to_mont(const uint8_t* in, uint32_t n, fr_t* out);   // n1.cu
__global__ void k_relu_range(const int32_t* Z, const int32_t* GA, uint64_t D, uint32_t QR, unsigned int* bad);

// the weights of Eq. (aux-Z) and of Z': s(j) = 2^j (j < QR-1), -2^(QR-1); s'(j) = [j = R-1] +
// 2^(j-R) (R <= j < QR-1) - 2^(Q-1) [j = QR-1]; zero for j >= QR
__device__ inline fr_t rs_s(uint32_t j, uint32_t QR) {
    if (j >= QR) return fr_zero();
    const fr_t v = fr_from_u32(1u << (j == QR - 1 ? QR - 1 : j));
    return j == QR - 1 ? fr_neg(v) : v;
}
__device__ inline fr_t rs_sp(uint32_t j, uint32_t Q, uint32_t R) {
    const uint32_t QR = Q + R;
    if (j >= QR || j + 1 < R) return fr_zero();
    if (j == R - 1) return fr_one();
    if (j == QR - 1) return fr_neg(fr_from_u32(1u << (Q - 1)));
    return fr_from_u32(1u << (j - R));
}

// W(i, j) = EZ[i] s(j) + EP[i] s'(j) (EZ already scaled by r), flat i * 2^logB + j
__global__ void k_rs_weights(const fr_t* EZ, const fr_t* EP, uint64_t D, uint32_t logB, uint32_t Q, uint32_t R, fr_t* W) {
    __shared__ fr_t sw[64];
    const uint32_t B = 1u << logB;
    if (threadIdx.x < B) {
        sw[threadIdx.x] = rs_s(threadIdx.x, Q + R);
        sw[32 + threadIdx.x] = rs_sp(threadIdx.x, Q, R);
    }
    __syncthreads();
    const uint64_t n = D << logB;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t j = (uint32_t)(x & (B - 1));
        const uint64_t i = x >> logB;
        fr_store(&W[x], fr_add(fr_mul(fr_load(&EZ[i]), sw[j]), fr_mul(fr_load(&EP[i]), sw[32 + j])));
    }
}

// aux bits (a) and a - 1 as int32 tables
__global__ void k_rs_bits(const int32_t* Z, uint64_t D, uint32_t logB, uint32_t QR, int32_t* a, int32_t* am1) {
    const uint64_t n = D << logB;
    const LoadBits L{Z, logB, QR};
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) {
        const int32_t v = L(x);
        a[x] = v;
        am1[x] = v - 1;
    }
}

// claim of A: r c_Z + c_P
__global__ void k_rs_claim(const fr_t* r, const fr_t* cl, fr_t* out) {
    fr_store(out, fr_add(fr_mul_cold(fr_load(r), fr_load(&cl[0])), fr_load(&cl[1])));
}

}  // namespace zk

extern "C" {

zk_status zk_hadamard_zero_prove(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_Y, const int32_t* d_A,
                                 const int32_t* d_B, uint32_t m, uint8_t* proof, uint64_t* proof_len, zk_fr* w_out,
                                 zk_fr* point_out, zk_fr* finals_out) {
    if (!ctx) return ZK_ERR_ARG;
    try {
        ZK_CUDA(cudaSetDevice(ctx->device));
        ZK_REQUIRE(tr && d_Y && d_A && d_B && m >= 1 && m <= 34, ZK_ERR_ARG, "bad zero-form statement");
        const uint64_t plen = 4 + 32ull * 3 * m + 96;   // u32le m | m x 3 evaluations | Y~, A~, B~ at r
        if (proof_len) {
            const bool query = !proof;
            if (proof && *proof_len < plen) {
                *proof_len = plen;
                throw ZkError{ZK_ERR_ARG, "proof buffer too small"};
            }
            *proof_len = plen;
            if (query) return ZK_OK;
        }
        Scratch s(ctx);
        uint8_t hdr[4] = {(uint8_t)m, (uint8_t)(m >> 8), (uint8_t)(m >> 16), (uint8_t)(m >> 24)};
        tr_absorb_host(tr, "hd/hdr", hdr, 4);
        fr_t* w = s.alloc<fr_t>(m);
        uint8_t* wc = s.alloc<uint8_t>(32ull * m);
        tr_challenges_dev(tr, "hd/w", m, w, wc);
        const uint64_t N = 1ull << m;
        ScEngine e;
        e.ctx = ctx;
        e.tr = tr;
        e.s = &s;
        e.m = m;
        e.n_eq = m;
        e.K = 3;
        e.zero = true;
        e.d_w = w;
        e.d_scale = nullptr;
        // the engine's proof layout: 44-byte head (unused here) | m x 3 evaluations | 3 finals
        uint8_t* d_proof = s.alloc<uint8_t>(44 + 32ull * 3 * m + 96);
        e.d_proof = d_proof;
        e.d_r = s.alloc<fr_t>(m);
        e.d_point = s.alloc<uint8_t>(32ull * m);
        e.d_claim = s.alloc_zero<fr_t>(1);
        e.claim_given = true;
        e.d_finals = nullptr;
        const fr_t* tabs[3] = {s.alloc<fr_t>(N), s.alloc<fr_t>(N), s.alloc<fr_t>(N)};
        const int32_t* i32[3] = {d_Y, d_A, d_B};
        e.setup(tabs, m, 0, m);
        e.set_i32(i32);
        e.run_to_end();
        if (proof) {
            std::memcpy(proof, hdr, 4);
            ZK_CUDA(cudaMemcpyAsync(proof + 4, d_proof + 44, plen - 4, cudaMemcpyDeviceToHost, ctx->stream));
        }
        if (w_out) ZK_CUDA(cudaMemcpyAsync(w_out, wc, 32ull * m, cudaMemcpyDeviceToHost, ctx->stream));
        if (point_out) ZK_CUDA(cudaMemcpyAsync(point_out, e.d_point, 32ull * m, cudaMemcpyDeviceToHost, ctx->stream));
        if (finals_out)
            ZK_CUDA(cudaMemcpyAsync(finals_out, d_proof + 44 + 32ull * 3 * m, 96, cudaMemcpyDeviceToHost, ctx->stream));
        ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (const ZkError& err) {
        ctx->err = err.msg;
        return err.st;
    } catch (const std::exception& err) {
        ctx->err = err.what();
        return ZK_ERR_INTERNAL;
    }
    return ZK_OK;
}

// The loss-gradient family, Eq. (fcnn-GZ-last) P:L299-302 (D24): G_Z = Z - Y is linear, so at the
// verifier's point u the claims G_Z~(u), Z~(u), Y~(u) (lazy int32 MLEs, mle_i32_plain) close it.
zk_status zk_loss_grad_prove(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_GZ, const int32_t* d_Z,
                             const int32_t* d_Y, uint32_t m, zk_fr* point_out, zk_fr* claims_out) {
    if (!ctx) return ZK_ERR_ARG;
    try {
        ZK_CUDA(cudaSetDevice(ctx->device));
        ZK_REQUIRE(tr && d_GZ && d_Z && d_Y && m >= 1 && m <= 34, ZK_ERR_ARG, "bad loss-gradient statement");
        Scratch s(ctx);
        uint8_t hdr[4] = {(uint8_t)m, (uint8_t)(m >> 8), (uint8_t)(m >> 16), (uint8_t)(m >> 24)};
        tr_absorb_host(tr, "lg/hdr", hdr, 4);
        fr_t* u = s.alloc<fr_t>(m);
        uint8_t* uc = s.alloc<uint8_t>(32ull * m);
        tr_challenges_dev(tr, "lg/u", m, u, uc);
        fr_t* cl = s.alloc<fr_t>(3);
        mle_i32_plain(ctx, d_GZ, m, u, cl, s);
        mle_i32_plain(ctx, d_Z, m, u, cl + 1, s);
        mle_i32_plain(ctx, d_Y, m, u, cl + 2, s);
        uint8_t* cc = s.alloc<uint8_t>(96);
        to_canonical_dev(ctx, cl, 3, cc);
        ZK_LAUNCH(ctx, k_tr_absorb_dev, 1, 32, 0, tr->d_st, make_tag("lg/claims"), (const uint8_t*)cc, (uint64_t)96);
        if (point_out) ZK_CUDA(cudaMemcpyAsync(point_out, uc, 32ull * m, cudaMemcpyDeviceToHost, ctx->stream));
        if (claims_out) ZK_CUDA(cudaMemcpyAsync(claims_out, cc, 96, cudaMemcpyDeviceToHost, ctx->stream));
        ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (const ZkError& err) {
        ctx->err = err.msg;
        return err.st;
    } catch (const std::exception& err) {
        ctx->err = err.what();
        return ZK_ERR_INTERNAL;
    }
    return ZK_OK;
}

// The loss-gradient family with device outputs: d_out = u (m canonical) | the three claims (canonical).
zk_status zk_loss_grad_prove_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_GZ, const int32_t* d_Z,
                                 const int32_t* d_Y, uint32_t m, uint8_t* d_out, uint64_t* out_len) {
    if (!ctx) return ZK_ERR_ARG;
    try {
        ZK_CUDA(cudaSetDevice(ctx->device));
        const uint64_t need = 32ull * m + 96;
        ZK_REQUIRE(d_out || out_len, ZK_ERR_ARG, "null output");
        if (!d_out) {
            *out_len = need;
            return ZK_OK;
        }
        ZK_REQUIRE(out_len && *out_len >= need, ZK_ERR_ARG, "d_out too small (*out_len < the required size)");
        *out_len = need;
        ZK_REQUIRE(tr && d_GZ && d_Z && d_Y && m >= 1 && m <= 34, ZK_ERR_ARG, "bad loss-gradient statement");
        Scratch s(ctx);
        uint8_t hdr[4] = {(uint8_t)m, (uint8_t)(m >> 8), (uint8_t)(m >> 16), (uint8_t)(m >> 24)};
        tr_absorb_host(tr, "lg/hdr", hdr, 4);
        fr_t* u = s.alloc<fr_t>(m);
        tr_challenges_dev(tr, "lg/u", m, u, d_out);
        fr_t* cl = s.alloc<fr_t>(3);
        mle_i32_plain(ctx, d_GZ, m, u, cl, s);
        mle_i32_plain(ctx, d_Z, m, u, cl + 1, s);
        mle_i32_plain(ctx, d_Y, m, u, cl + 2, s);
        to_canonical_dev(ctx, cl, 3, d_out + 32ull * m);
        ZK_LAUNCH(ctx, k_tr_absorb_dev, 1, 32, 0, tr->d_st, make_tag("lg/claims"), (const uint8_t*)(d_out + 32ull * m),
                  (uint64_t)96);
    } catch (const ZkError& err) {
        ctx->err = err.msg;
        return err.st;
    } catch (const std::exception& err) {
        ctx->err = err.what();
        return ZK_ERR_INTERNAL;
    }
    return ZK_OK;
}

// The top-layer rescale (D26): claims Z~(u_Z), Z'~(u_P) at the given points, then the two product
// sumchecks over the bits of Z (A: the weighted reconstruction, B: the bits are binary).
zk_status zk_rescale_prove_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_Z, uint32_t logD, uint32_t Q,
                               uint32_t R, const uint8_t* d_pts, uint8_t* d_out, uint64_t* out_len,
                               uint32_t* d_range_flag) {
    if (!ctx) return ZK_ERR_ARG;
    try {
        ZK_CUDA(cudaSetDevice(ctx->device));
        ZK_REQUIRE(Q >= 1 && R >= 1 && Q <= 32 && R <= 32 && Q + R <= 32 && logD >= 1 && logD <= 26, ZK_ERR_ARG,
                   "bad rescale shape");
        const uint32_t QR = Q + R;
        uint32_t logB = 0;
        while ((1u << logB) < QR) logB++;
        const uint32_t m = logB + logD;
        const uint64_t D = 1ull << logD, n = 1ull << m;
        const uint64_t lp = sumcheck_proof_len(m, 2);
        const uint64_t plen = 12 + 64 + 2 * lp, off_pa = (plen + 15) & ~15ull, need = off_pa + 64ull * m;
        ZK_REQUIRE(d_out || out_len, ZK_ERR_ARG, "null output");
        if (!d_out) {
            *out_len = need;
            return ZK_OK;
        }
        ZK_REQUIRE(out_len && *out_len >= need, ZK_ERR_ARG, "d_out too small (*out_len < the required size)");
        *out_len = need;
        ZK_REQUIRE(((uintptr_t)d_out & 15) == 0, ZK_ERR_ARG, "d_out must be 16-byte aligned");
        ZK_REQUIRE(tr && d_Z && d_pts && d_range_flag, ZK_ERR_ARG, "null argument");
        Scratch s(ctx);
        if (QR < 32) ZK_LAUNCH(ctx, k_relu_range, grid_for(ctx, D, 256, 8), 256, 0, d_Z, d_Z, D, QR, d_range_flag);
        uint8_t hdr[12];
        const uint32_t hv[3] = {logD, Q, R};
        for (int i = 0; i < 3; i++)
            for (int k = 0; k < 4; k++) hdr[4 * i + k] = (uint8_t)(hv[i] >> (8 * k));
        tr_absorb_host(tr, "rs/hdr", hdr, 12, d_out);
        fr_t* U = s.alloc<fr_t>(2ull * logD);
        ZK_LAUNCH(ctx, k_canon_to_mont, 1, 64, 0, d_pts, 2 * logD, U);
        fr_t* cl = s.alloc<fr_t>(2);
        mle_i32_plain(ctx, d_Z, logD, U, cl, s);
        mle_i32_relu(ctx, 2, d_Z, nullptr, R, logD, U + logD, cl + 1, s);
        ZK_LAUNCH(ctx, k_tr_absorb_frs, 1, 32, 0, tr->d_st, make_tag("rs/claims"), (const fr_t*)cl, 2u, d_out + 12);
        fr_t* r = s.alloc<fr_t>(1);
        tr_challenges_dev(tr, "rs/r", 1, r, nullptr);
        // A: W and the bits
        fr_t* EZ = s.alloc<fr_t>(D);
        fr_t* EP = s.alloc<fr_t>(D);
        eq_table_dev(ctx, U, logD, r, EZ, s);
        eq_table_dev(ctx, U + logD, logD, nullptr, EP, s);
        fr_t* W = s.alloc<fr_t>(n);
        ZK_LAUNCH(ctx, k_rs_weights, grid_for(ctx, n, 256, 8), 256, 0, (const fr_t*)EZ, (const fr_t*)EP, D, logB, Q, R, W);
        int32_t* a = s.alloc<int32_t>(n);
        int32_t* am1 = s.alloc<int32_t>(n);
        ZK_LAUNCH(ctx, k_rs_bits, grid_for(ctx, n, 256, 8), 256, 0, d_Z, D, logB, QR, a, am1);
        ScStatement A;
        memset(&A, 0, sizeof A);
        A.m = m;
        A.K = 2;
        A.tables[0] = W;
        A.tables[1] = s.alloc<fr_t>(n);
        A.i32[1] = a;
        A.d_claim = s.alloc<fr_t>(1);
        A.claim_given = true;
        ZK_LAUNCH(ctx, k_rs_claim, 1, 1, 0, (const fr_t*)r, (const fr_t*)cl, A.d_claim);
        A.d_proof = d_out + 76;
        A.d_r = s.alloc<fr_t>(m);
        A.d_point = d_out + off_pa;
        sumcheck_prove_dev(ctx, tr, A, s);
        // B: the bits are binary, sum_x beta(w, x) a(x) (a(x) - 1) = 0
        fr_t* w = s.alloc<fr_t>(m);
        tr_challenges_dev(tr, "rs/w", m, w, nullptr);
        ScStatement B;
        memset(&B, 0, sizeof B);
        B.m = m;
        B.n_eq = m;
        B.K = 2;
        B.tables[0] = s.alloc<fr_t>(n);
        B.tables[1] = s.alloc<fr_t>(n);
        B.i32[0] = a;
        B.i32[1] = am1;
        B.d_w = w;
        B.d_claim = s.alloc_zero<fr_t>(1);
        B.claim_given = true;
        B.d_proof = d_out + 76 + lp;
        B.d_r = s.alloc<fr_t>(m);
        B.d_point = d_out + off_pa + 32ull * m;
        sumcheck_prove_dev(ctx, tr, B, s);
    } catch (const ZkError& err) {
        ctx->err = err.msg;
        return err.st;
    } catch (const std::exception& err) {
        ctx->err = err.what();
        return ZK_ERR_INTERNAL;
    }
    return ZK_OK;
}

}  // extern "C"
