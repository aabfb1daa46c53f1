// n2.cu — SURVEY §8(f) N2: Protocol 2's zero form for the aggregated Hadamard product (Eq. tensor-op-aggr
// P:L229-234, Protocol 2 P:L476-502; D22), on the product-sumcheck engine (rows a4-a6)
// with the zero-form round kernel k_sc_zero_round; and the loss-gradient family (Eq. fcnn-GZ-last, D24).
#include <cstring>

#include "sumcheck.cuh"
#include "tables.cuh"

using namespace zk;

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

}  // extern "C"
