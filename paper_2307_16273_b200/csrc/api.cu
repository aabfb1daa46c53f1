// api.cu — the C ABI of libzkdl (include/zkdl.h): argument checking, marshalling, status codes.
#include <cstring>

#include "matmul.cuh"
#include "relu.cuh"
#include "sumcheck.cuh"
#include "tables.cuh"

using namespace zk;

namespace zk {
__global__ void k_from_canonical(const fr_t* in, uint64_t n, fr_t* out, unsigned int* bad);
void tr_init_dev(zk_transcript* tr, const uint8_t seed[32]);
void tr_fork_dev(zk_transcript* parent, const char* tag, uint8_t* d_child_st);
void tr_absorb_state_dev(zk_transcript* tr, const char* tag, const uint8_t* d_other_st);
void selftest_op_dev(zk_ctx* ctx, int op, const fr_t* a, const fr_t* b, uint64_t n, fr_t* out);
void mul_bench_dev(zk_ctx* ctx, const fr_t* seed, uint32_t iters, uint32_t blocks, fr_t* out);
}

#define ZK_API_BEGIN(ctx)                                                                              \
    if (!(ctx)) return ZK_ERR_ARG;                                                                     \
    try {                                                                                              \
        ZK_CUDA(cudaSetDevice((ctx)->device));
#define ZK_API_END(ctx)                                                                                \
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

const char* zk_version(void) { return "zkdl-b200 0.1 (sm_100a)"; }

zk_status zk_ctx_create(int device, void* cuda_stream, zk_ctx** out) {
    if (!out) return ZK_ERR_ARG;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0) return ZK_ERR_CUDA;
    if (cudaSetDevice(device) != cudaSuccess) return ZK_ERR_CUDA;
    int major = 0, sms = 0;   // (two attribute queries: cudaGetDeviceProperties costs milliseconds)
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
        return ZK_ERR_CUDA;
    if (major != 10) return ZK_ERR_CUDA;   // built for sm_100a only
    zk_ctx* c = new zk_ctx();
    c->device = device;
    c->stream = (cudaStream_t)cuda_stream;
    c->num_sms = sms;
    // keep freed scratch in the pool (no release back to the OS between calls)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    *out = c;
    return ZK_OK;
}

void zk_ctx_destroy(zk_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    zk_ctx_detach_nccl(ctx);
    if (ctx->aux) {
        cudaStreamSynchronize(ctx->aux);
        cudaStreamDestroy(ctx->aux);
        cudaEventDestroy(ctx->aux_ev[0]);
        cudaEventDestroy(ctx->aux_ev[1]);
    }
    delete ctx;
}

const char* zk_last_error(const zk_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
uint64_t zk_ctx_launch_count(const zk_ctx* ctx) { return ctx ? ctx->launches : 0; }

zk_status zk_ctx_synchronize(zk_ctx* ctx) {
    ZK_API_BEGIN(ctx)
    ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    ZK_API_END(ctx)
}

zk_status zk_ctx_set_sm_budget(zk_ctx* ctx, uint32_t sms) {
    ZK_API_BEGIN(ctx)
    ctx->sm_budget = (int)sms;
    ZK_API_END(ctx)
}

zk_status zk_ctx_set_persistent(zk_ctx* ctx, int allow) {
    ZK_API_BEGIN(ctx)
    ctx->no_persist = !allow;
    ZK_API_END(ctx)
}

zk_status zk_ctx_profile(zk_ctx* ctx, int enable) {
    ZK_API_BEGIN(ctx)
    ctx->prof = enable != 0;
    ZK_API_END(ctx)
}

zk_status zk_ctx_profile_filter(zk_ctx* ctx, const char* prefix) {
    ZK_API_BEGIN(ctx)
    ctx->prof_filter = prefix ? prefix : "";
    ZK_API_END(ctx)
}

zk_status zk_ctx_profile_read(zk_ctx* ctx, char* out, uint64_t cap) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(out && cap, ZK_ERR_ARG, "null buffer");
    ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    struct Agg {
        std::string name;
        uint64_t n;
        double ms;
    };
    std::vector<Agg> agg;
    for (auto& r : ctx->recs) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        bool found = false;
        for (auto& g : agg)
            if (g.name == r.name) {
                g.n++;
                g.ms += ms;
                found = true;
                break;
            }
        if (!found) agg.push_back({r.name, 1, (double)ms});
        ctx->ev_pool.push_back(r.a);
        ctx->ev_pool.push_back(r.b);
    }
    ctx->recs.clear();
    std::string s;
    char line[512];
    for (auto& g : agg) {
        snprintf(line, sizeof line, "%s\t%llu\t%.6f\n", g.name.c_str(), (unsigned long long)g.n, g.ms);
        s += line;
    }
    ZK_REQUIRE(s.size() + 1 <= cap, ZK_ERR_ARG, "profile buffer too small");
    memcpy(out, s.c_str(), s.size() + 1);
    ZK_API_END(ctx)
}

// ------------------------------------------------------------------ transcript
zk_status zk_transcript_new(zk_ctx* ctx, const uint8_t seed[32], zk_transcript** out) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(seed && out, ZK_ERR_ARG, "null argument");
    zk_transcript* t = new zk_transcript();
    t->ctx = ctx;
    cudaError_t e = cudaMallocAsync(&t->d_st, 32, ctx->stream);   // stream-ordered: no synchronisation
    if (e != cudaSuccess) {
        delete t;
        throw ZkError{ZK_ERR_OOM, "cudaMallocAsync transcript"};
    }
    tr_init_dev(t, seed);
    *out = t;
    ZK_API_END(ctx)
}

zk_status zk_transcript_absorb(zk_transcript* tr, const char* tag, const void* msg, uint64_t len) {
    if (!tr) return ZK_ERR_ARG;
    zk_ctx* ctx = tr->ctx;
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(tag && (msg || !len), ZK_ERR_ARG, "null argument");
    tr_absorb_host(tr, tag, msg, len);
    ZK_API_END(ctx)
}

zk_status zk_transcript_challenges(zk_transcript* tr, const char* tag, uint32_t n, zk_fr* out) {
    if (!tr) return ZK_ERR_ARG;
    zk_ctx* ctx = tr->ctx;
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(tag && (out || !n), ZK_ERR_ARG, "null argument");
    if (!n) return ZK_OK;
    Scratch s(ctx);
    uint8_t* d = s.alloc<uint8_t>(32ull * n);
    tr_challenges_dev(tr, tag, n, nullptr, d);
    ZK_CUDA(cudaMemcpyAsync(out, d, 32ull * n, cudaMemcpyDeviceToHost, ctx->stream));
    ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    ZK_API_END(ctx)
}

zk_status zk_transcript_state(zk_transcript* tr, uint8_t out[32]) {
    if (!tr || !out) return ZK_ERR_ARG;
    zk_ctx* ctx = tr->ctx;
    ZK_API_BEGIN(ctx)
    ZK_CUDA(cudaMemcpyAsync(out, tr->d_st, 32, cudaMemcpyDeviceToHost, ctx->stream));
    ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    ZK_API_END(ctx)
}

zk_status zk_transcript_fork(zk_transcript* parent, const char* tag, zk_ctx* child_ctx, zk_transcript** out) {
    if (!parent) return ZK_ERR_ARG;
    zk_ctx* ctx = parent->ctx;
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(tag && out, ZK_ERR_ARG, "null argument");
    zk_transcript* t = new zk_transcript();
    t->ctx = child_ctx ? child_ctx : ctx;
    cudaError_t e = cudaMallocAsync(&t->d_st, 32, ctx->stream);   // written on the parent's stream
    if (e != cudaSuccess) {
        delete t;
        throw ZkError{ZK_ERR_OOM, "cudaMallocAsync transcript"};
    }
    try {
        tr_fork_dev(parent, tag, t->d_st);
    } catch (...) {
        cudaFreeAsync(t->d_st, ctx->stream);
        delete t;
        throw;
    }
    *out = t;
    ZK_API_END(ctx)
}

zk_status zk_transcript_absorb_state(zk_transcript* tr, const char* tag, const zk_transcript* other) {
    if (!tr || !other) return ZK_ERR_ARG;
    zk_ctx* ctx = tr->ctx;
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(tag, ZK_ERR_ARG, "null tag");
    tr_absorb_state_dev(tr, tag, other->d_st);
    ZK_API_END(ctx)
}

void zk_transcript_free(zk_transcript* tr) {
    if (!tr) return;
    cudaSetDevice(tr->ctx->device);
    cudaFreeAsync(tr->d_st, tr->ctx->stream);   // after every enqueued use of the state
    delete tr;
}

// ------------------------------------------------------------------ tables
zk_status zk_embed_i32(zk_ctx* ctx, const int32_t* d_in, uint64_t n, void* d_out) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE((d_in && d_out) || !n, ZK_ERR_ARG, "null argument");
    embed_i32_dev(ctx, d_in, n, static_cast<fr_t*>(d_out));
    ZK_API_END(ctx)
}

// int16 -> int32 (the end-to-end transport of small-range stacks: half the host-to-device bytes)
__global__ void k_widen_i16(const int16_t* in, uint64_t n, int32_t* out) {
    const uint64_t n8 = n / 8;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n8; i += (uint64_t)gridDim.x * blockDim.x) {
        const int4 v = __ldcs(reinterpret_cast<const int4*>(in) + i);
        const int16_t* h = reinterpret_cast<const int16_t*>(&v);
        int4* o = reinterpret_cast<int4*>(out) + 2 * i;
        __stcs(o, make_int4(h[0], h[1], h[2], h[3]));
        __stcs(o + 1, make_int4(h[4], h[5], h[6], h[7]));
    }
    for (uint64_t i = 8 * n8 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

// out[s][e] = base[s][e] (s < L), out[s][e] = out[s - L][e] + delta[s - L][e] (L <= s < n_slots): one thread per
// (l < L, 4 consecutive entries), walking its slots l, l + L, ... (4 B of deltas in, 16 B out per slot step)
__global__ void k_undelta_i8(const int16_t* base, const int8_t* delta, uint64_t slot, uint32_t L, uint32_t n_slots,
                             int32_t* out) {
    const uint64_t q = slot / 4, total = q * L;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t l = (uint32_t)(i / q);
        const uint64_t e = 4 * (i % q);
        const short2 b0 = *reinterpret_cast<const short2*>(base + (uint64_t)l * slot + e);
        const short2 b1 = *reinterpret_cast<const short2*>(base + (uint64_t)l * slot + e + 2);
        int4 v = make_int4(b0.x, b0.y, b1.x, b1.y);
        __stcs(reinterpret_cast<int4*>(out + (uint64_t)l * slot + e), v);
        for (uint32_t s = l + L; s < n_slots; s += L) {
            const char4 d = __ldcs(reinterpret_cast<const char4*>(delta + (uint64_t)(s - L) * slot + e));
            v.x += d.x;
            v.y += d.y;
            v.z += d.z;
            v.w += d.w;
            __stcs(reinterpret_cast<int4*>(out + (uint64_t)s * slot + e), v);
        }
    }
}

zk_status zk_undelta_i8(zk_ctx* ctx, const int16_t* d_base, const int8_t* d_delta, uint64_t slot_elems, uint32_t L,
                        uint32_t n_slots, int32_t* d_out) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(d_base && d_out && L >= 1 && n_slots >= L && (d_delta || n_slots == L), ZK_ERR_ARG, "bad argument");
    ZK_REQUIRE(slot_elems % 4 == 0 && ((uintptr_t)d_out & 15) == 0 && ((uintptr_t)d_base & 7) == 0 &&
                   ((uintptr_t)d_delta & 3) == 0,
               ZK_ERR_ARG, "slot_elems must be a multiple of 4, buffers aligned (out 16, base 8, delta 4 bytes)");
    if (slot_elems)
        ZK_LAUNCH(ctx, k_undelta_i8, grid_for(ctx, slot_elems / 4 * L, 256, 8), 256, 0, d_base, d_delta, slot_elems, L,
                  n_slots, d_out);
    ZK_API_END(ctx)
}

zk_status zk_widen_i16(zk_ctx* ctx, const int16_t* d_in, uint64_t n, int32_t* d_out) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE((d_in && d_out) || !n, ZK_ERR_ARG, "null argument");
    ZK_REQUIRE(((uintptr_t)d_in & 15) == 0 && ((uintptr_t)d_out & 15) == 0, ZK_ERR_ARG, "buffers must be 16-byte aligned");
    if (n) ZK_LAUNCH(ctx, k_widen_i16, grid_for(ctx, (n + 7) / 8, 256, 8), 256, 0, d_in, n, d_out);
    ZK_API_END(ctx)
}

zk_status zk_eq_table(zk_ctx* ctx, const zk_fr* point, uint32_t k, const zk_fr* scale, void* d_out) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(d_out && (point || !k) && k <= 32, ZK_ERR_ARG, "bad argument");
    Scratch s(ctx);
    fr_t* u = s.alloc<fr_t>(k ? k : 1);
    upload_points(ctx, point, k, u, s);
    fr_t* sc = nullptr;
    if (scale) {
        sc = s.alloc<fr_t>(1);
        upload_points(ctx, scale, 1, sc, s);
    }
    eq_table_dev(ctx, u, k, sc, static_cast<fr_t*>(d_out), s);
    ZK_API_END(ctx)
}

zk_status zk_mle_eval_i32(zk_ctx* ctx, const int32_t* d_tab, uint32_t m, const zk_fr* point, zk_fr* out) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(d_tab && out && (point || !m) && m <= 40, ZK_ERR_ARG, "bad argument");
    Scratch s(ctx);
    fr_t* u = s.alloc<fr_t>(m ? m : 1);
    upload_points(ctx, point, m, u, s);
    fr_t* r = s.alloc<fr_t>(1);
    mle_i32_plain(ctx, d_tab, m, u, r, s);
    to_canonical_dev(ctx, r, 1, reinterpret_cast<uint8_t*>(r));
    ZK_CUDA(cudaMemcpyAsync(out, r, 32, cudaMemcpyDeviceToHost, ctx->stream));
    ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    ZK_API_END(ctx)
}

zk_status zk_mle_eval_fr(zk_ctx* ctx, const void* d_tab, uint32_t m, const zk_fr* point, zk_fr* out) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(d_tab && out && (point || !m) && m <= 40, ZK_ERR_ARG, "bad argument");
    Scratch s(ctx);
    fr_t* u = s.alloc<fr_t>(m ? m : 1);
    upload_points(ctx, point, m, u, s);
    fr_t* r = s.alloc<fr_t>(1);
    mle_fr_dev(ctx, static_cast<const fr_t*>(d_tab), m, u, r, s);
    to_canonical_dev(ctx, r, 1, reinterpret_cast<uint8_t*>(r));
    ZK_CUDA(cudaMemcpyAsync(out, r, 32, cudaMemcpyDeviceToHost, ctx->stream));
    ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    ZK_API_END(ctx)
}

zk_status zk_fr_table_to_canonical(zk_ctx* ctx, const void* d_in, uint64_t n, void* d_out) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE((d_in && d_out) || !n, ZK_ERR_ARG, "null argument");
    to_canonical_dev(ctx, static_cast<const fr_t*>(d_in), n, static_cast<uint8_t*>(d_out));
    ZK_API_END(ctx)
}

zk_status zk_fr_table_from_canonical(zk_ctx* ctx, const void* d_in, uint64_t n, void* d_out) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE((d_in && d_out) || !n, ZK_ERR_ARG, "null argument");
    if (!n) return ZK_OK;
    Scratch s(ctx);
    unsigned int* bad = s.alloc_zero<unsigned int>(1);
    ZK_LAUNCH(ctx, k_from_canonical, grid_for(ctx, n, 256, 8), 256, 0, static_cast<const fr_t*>(d_in), n,
              static_cast<fr_t*>(d_out), bad);
    unsigned int hbad = 0;
    ZK_CUDA(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, ctx->stream));
    ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    ZK_REQUIRE(!hbad, ZK_ERR_NONCANONICAL, "table entry >= p");
    ZK_API_END(ctx)
}

// ------------------------------------------------------------------ matmul
zk_status zk_matmul_reduce(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_A, const int32_t* d_B, zk_mm_shape shape,
                           void* d_At, void* d_Bt, zk_fr* point_out, zk_fr* claim_out) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(tr && d_A && d_B && d_At && d_Bt, ZK_ERR_ARG, "null argument");
    Scratch s(ctx);
    const uint32_t np = shape.logN + shape.logD1 + shape.logD3;
    fr_t* pts = s.alloc<fr_t>(np ? np : 1);
    uint8_t* pts_c = s.alloc<uint8_t>(32ull * (np ? np : 1) + 32);
    fr_t* claim = s.alloc<fr_t>(1);
    matmul_reduce_dev(ctx, tr, d_A, d_B, shape, static_cast<fr_t*>(d_At), static_cast<fr_t*>(d_Bt), pts, pts_c, claim, s);
    to_canonical_dev(ctx, claim, 1, pts_c + 32ull * np);
    if (point_out && np) ZK_CUDA(cudaMemcpyAsync(point_out, pts_c, 32ull * np, cudaMemcpyDeviceToHost, ctx->stream));
    if (claim_out) ZK_CUDA(cudaMemcpyAsync(claim_out, pts_c + 32ull * np, 32, cudaMemcpyDeviceToHost, ctx->stream));
    ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    ZK_API_END(ctx)
}

// ------------------------------------------------------------------ product sumcheck
zk_status zk_sumcheck_prove(zk_ctx* ctx, zk_transcript* tr, const zk_prod_stmt* st, void* const* d_tables,
                            const zk_fr* claim, zk_fr* claim_out, uint8_t* proof, uint64_t* proof_len, zk_fr* point_out,
                            zk_fr* finals_out) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(tr && st && d_tables, ZK_ERR_ARG, "null argument");
    const uint32_t m = st->m, n_eq = st->n_eq, K = st->n_tables;
    ZK_REQUIRE(m >= 1 && m <= 40 && n_eq <= m && K >= 1 && K <= 3, ZK_ERR_ARG, "bad statement");
    ZK_REQUIRE(st->w || !n_eq, ZK_ERR_ARG, "missing w");
    const uint64_t plen = sumcheck_proof_len(m, K);
    if (proof_len) {
        const bool query = !proof;
        if (proof && *proof_len < plen) {
            *proof_len = plen;
            throw ZkError{ZK_ERR_ARG, "proof buffer too small"};
        }
        *proof_len = plen;
        if (query) return ZK_OK;   // size query: nothing is proved, the transcript is untouched
    }
    for (uint32_t k = 0; k < K; k++) ZK_REQUIRE(d_tables[k], ZK_ERR_ARG, "null table");
    Scratch s(ctx);
    ScStatement S;
    memset(&S, 0, sizeof S);
    S.m = m;
    S.n_eq = n_eq;
    S.K = K;
    const uint64_t N = 1ull << m;
    for (uint32_t k = 0; k < K; k++) {
        if (st->i32_mask & (1u << k)) {   // embedded by the prover (fused into round 0 where it can)
            S.tables[k] = s.alloc<fr_t>(N);
            S.i32[k] = static_cast<const int32_t*>(d_tables[k]);
        } else {
            S.tables[k] = static_cast<const fr_t*>(d_tables[k]);
        }
    }
    fr_t* w = s.alloc<fr_t>(n_eq ? n_eq : 1);
    upload_points(ctx, st->w, n_eq, w, s);
    S.d_w = w;
    S.d_claim = s.alloc<fr_t>(1);
    if (claim) {
        upload_points(ctx, claim, 1, S.d_claim, s);
        S.claim_given = true;
    }
    S.d_proof = s.alloc<uint8_t>(plen);
    S.d_r = s.alloc<fr_t>(m);
    S.d_point = s.alloc<uint8_t>(32ull * m);
    S.d_finals = nullptr;
    sumcheck_prove_dev(ctx, tr, S, s);
    if (proof) ZK_CUDA(cudaMemcpyAsync(proof, S.d_proof, plen, cudaMemcpyDeviceToHost, ctx->stream));
    if (claim_out) ZK_CUDA(cudaMemcpyAsync(claim_out, S.d_proof + 12, 32, cudaMemcpyDeviceToHost, ctx->stream));
    if (point_out) ZK_CUDA(cudaMemcpyAsync(point_out, S.d_point, 32ull * m, cudaMemcpyDeviceToHost, ctx->stream));
    if (finals_out)
        ZK_CUDA(cudaMemcpyAsync(finals_out, S.d_proof + 44 + 32ull * m * (K + 1), 32ull * K, cudaMemcpyDeviceToHost,
                                ctx->stream));
    ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    ZK_API_END(ctx)
}

// ------------------------------------------------------------------ zkReLU
zk_status zk_relu_tables(zk_ctx* ctx, const int32_t* d_Z, const int32_t* d_GA, uint64_t D, uint32_t Q, uint32_t R,
                         uint8_t* d_sign, int32_t* d_A, int32_t* d_GZ, int32_t* d_Zp, int32_t* d_GAp, int32_t* d_RZ,
                         int32_t* d_RGA) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(d_Z && d_GA && d_sign && d_A && d_GZ, ZK_ERR_ARG, "null argument");
    ZK_REQUIRE(Q >= 1 && R >= 1 && Q <= 32 && R <= 32 && Q + R <= 32, ZK_ERR_ARG, "need 1 <= Q, R and Q + R <= 32");
    Scratch s(ctx);
    bool ok = relu_tables_dev(ctx, d_Z, d_GA, D, Q, R, d_sign, d_A, d_GZ, d_Zp, d_GAp, d_RZ, d_RGA, s);
    ZK_REQUIRE(ok, ZK_ERR_RANGE, "Z or G_A outside the (Q+R)-bit range");
    ZK_API_END(ctx)
}

zk_status zk_relu_prove(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_Z, const int32_t* d_GA, uint32_t logD,
                        uint32_t Q, uint32_t R, uint8_t* proof, uint64_t* proof_len, zk_fr* claims_out, zk_fr* point_out,
                        zk_fr* finals_out) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(tr && d_Z && d_GA, ZK_ERR_ARG, "null argument");
    ZK_REQUIRE(Q >= 1 && R >= 1 && Q <= 32 && R <= 32 && Q + R <= 32 && logD >= 1 && logD <= 30, ZK_ERR_ARG, "bad zkReLU shape");
    const uint32_t logB = relu_logB(Q, R);
    const uint64_t plen = relu_proof_len(logD, logB);
    if (proof_len) {
        const bool query = !proof;
        if (proof && *proof_len < plen) {
            *proof_len = plen;
            throw ZkError{ZK_ERR_ARG, "proof buffer too small"};
        }
        *proof_len = plen;
        if (query) return ZK_OK;   // size query: nothing is proved, the transcript is untouched
    }
    Scratch s(ctx);
    ReluOutputs o;
    o.d_proof = s.alloc<uint8_t>(plen);
    o.d_point = s.alloc<uint8_t>(32ull * (logB + logD));
    unsigned int* range_bad = s.alloc_zero<unsigned int>(1);
    relu_prove_dev(ctx, tr, d_Z, d_GA, logD, Q, R, o, range_bad, s);
    unsigned int hbad = 0;
    ZK_CUDA(cudaMemcpyAsync(&hbad, range_bad, 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (proof) ZK_CUDA(cudaMemcpyAsync(proof, o.d_proof, plen, cudaMemcpyDeviceToHost, ctx->stream));
    if (claims_out) ZK_CUDA(cudaMemcpyAsync(claims_out, o.d_proof + 12, 128, cudaMemcpyDeviceToHost, ctx->stream));
    if (point_out)
        ZK_CUDA(cudaMemcpyAsync(point_out, o.d_point, 32ull * (logB + logD), cudaMemcpyDeviceToHost, ctx->stream));
    if (finals_out)
        ZK_CUDA(cudaMemcpyAsync(finals_out, o.d_proof + plen - 96, 96, cudaMemcpyDeviceToHost, ctx->stream));
    ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    ZK_REQUIRE(!hbad, ZK_ERR_RANGE, "Z or G_A outside the (Q+R)-bit range");
    ZK_API_END(ctx)
}

// ------------------------------------------------------------------ device-output provers
// d_out == NULL: size query (*out_len = need).  Otherwise *out_len is the caller's capacity and must
// hold `need` bytes (else ZK_ERR_ARG, nothing written); on return it is the size written.
static bool size_query(uint8_t* d_out, uint64_t* out_len, uint64_t need) {
    ZK_REQUIRE(d_out || out_len, ZK_ERR_ARG, "null output");
    if (!d_out) {
        *out_len = need;
        return true;
    }
    ZK_REQUIRE(out_len, ZK_ERR_ARG, "out_len (the capacity of d_out) is required");
    ZK_REQUIRE(*out_len >= need, ZK_ERR_ARG, "d_out too small (*out_len < the required size)");
    *out_len = need;
    return false;
}

zk_status zk_matmul_prove(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_A, const int32_t* d_B, zk_mm_shape shape,
                          void* d_At, void* d_Bt, uint8_t* d_out, uint64_t* out_len) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(tr && d_A && d_B, ZK_ERR_ARG, "null argument");
    const uint32_t np = shape.logN + shape.logD1 + shape.logD3;
    const uint32_t m = shape.logN + shape.logD2, K = 2;
    const uint64_t plen = sumcheck_proof_len(m, K);
    const uint64_t off_proof = 32ull * np + 32, off_r = (off_proof + plen + 15) & ~15ull;
    if (size_query(d_out, out_len, off_r + 32ull * m)) return ZK_OK;
    ZK_REQUIRE(m >= 1 && m <= 40, ZK_ERR_ARG, "bad matmul shape");
    ZK_REQUIRE(((uintptr_t)d_out & 15) == 0, ZK_ERR_ARG, "d_out must be 16-byte aligned");
    Scratch s(ctx);
    const uint64_t N = 1ull << m;
    fr_t* At = d_At ? static_cast<fr_t*>(d_At) : s.alloc<fr_t>(N);
    fr_t* Bt = d_Bt ? static_cast<fr_t*>(d_Bt) : s.alloc<fr_t>(N);
    fr_t* pts = s.alloc<fr_t>(np ? np : 1);
    fr_t* claim = s.alloc<fr_t>(1);
    matmul_reduce_dev(ctx, tr, d_A, d_B, shape, At, Bt, pts, d_out, claim, s);
    to_canonical_dev(ctx, claim, 1, d_out + 32ull * np);
    ScStatement S;
    memset(&S, 0, sizeof S);
    S.m = m;
    S.n_eq = shape.logN;
    S.K = K;
    S.tables[0] = At;
    S.tables[1] = Bt;
    S.d_w = pts;   // w = the first logN entries of the point
    S.d_claim = claim;
    S.claim_given = true;
    S.d_proof = d_out + off_proof;
    S.d_r = s.alloc<fr_t>(m);
    S.d_point = d_out + off_r;
    S.d_finals = nullptr;
    sumcheck_prove_dev(ctx, tr, S, s);
    ZK_API_END(ctx)
}

static zk_status relu_prove_dev_entry(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_Z, const int32_t* d_GA, uint32_t logD,
                            uint32_t Q, uint32_t R, uint8_t* d_out, uint64_t* out_len, uint32_t* d_range_flag, const uint8_t* d_pts) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(tr && d_Z && d_GA && d_range_flag, ZK_ERR_ARG, "null argument");
    ZK_REQUIRE(Q >= 1 && R >= 1 && Q <= 32 && R <= 32 && Q + R <= 32 && logD >= 1 && logD <= 30, ZK_ERR_ARG, "bad zkReLU shape");
    const uint32_t logB = relu_logB(Q, R);
    const uint64_t plen = relu_proof_len(logD, logB);
    const uint64_t off_pt = (plen + 15) & ~15ull;
    if (size_query(d_out, out_len, off_pt + 32ull * (logB + logD))) return ZK_OK;
    ZK_REQUIRE(((uintptr_t)d_out & 15) == 0, ZK_ERR_ARG, "d_out must be 16-byte aligned");
    Scratch s(ctx);
    ReluOutputs o;
    o.d_proof = d_out;
    o.d_point = d_out + off_pt;
    relu_prove_dev(ctx, tr, d_Z, d_GA, logD, Q, R, o, d_range_flag, s, d_pts);
    ZK_API_END(ctx)
}

zk_status zk_relu_prove_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_Z, const int32_t* d_GA, uint32_t logD,
                            uint32_t Q, uint32_t R, uint8_t* d_out, uint64_t* out_len, uint32_t* d_range_flag) {
    return relu_prove_dev_entry(ctx, tr, d_Z, d_GA, logD, Q, R, d_out, out_len, d_range_flag, nullptr);
}

zk_status zk_relu_prove_chained_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_Z, const int32_t* d_GA,
                                    uint32_t logD, uint32_t Q, uint32_t R, const uint8_t* d_pts, uint8_t* d_out,
                                    uint64_t* out_len, uint32_t* d_range_flag) {
    if (!d_pts && d_out) return ZK_ERR_ARG;
    return relu_prove_dev_entry(ctx, tr, d_Z, d_GA, logD, Q, R, d_out, out_len, d_range_flag, d_pts);
}

zk_status zk_transcript_state_dev(zk_transcript* tr, void* d_out) {
    if (!tr || !d_out) return ZK_ERR_ARG;
    zk_ctx* ctx = tr->ctx;
    ZK_API_BEGIN(ctx)
    ZK_CUDA(cudaMemcpyAsync(d_out, tr->d_st, 32, cudaMemcpyDeviceToDevice, ctx->stream));
    ZK_API_END(ctx)
}

// ------------------------------------------------------------------ diagnostics (tests and the Fr-mul peak probe)
zk_status zk_diag_fr_op(zk_ctx* ctx, int op, const void* d_a, const void* d_b, uint64_t n, void* d_out) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(d_a && d_out && op >= 0 && op <= 6, ZK_ERR_ARG, "bad argument");
    selftest_op_dev(ctx, op, static_cast<const fr_t*>(d_a), static_cast<const fr_t*>(d_b), n, static_cast<fr_t*>(d_out));
    ZK_API_END(ctx)
}

zk_status zk_diag_rowdot(zk_ctx* ctx, const int32_t* d_M, uint64_t nrows, uint32_t cols, const zk_fr* point,
                         void* d_out, int use_tc) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(d_M && d_out && point && cols && (cols & (cols - 1)) == 0, ZK_ERR_ARG, "bad argument");
    uint32_t k = 0;
    while ((1u << k) < cols) k++;
    Scratch s(ctx);
    fr_t* u = s.alloc<fr_t>(k ? k : 1);
    if (k) upload_points(ctx, point, k, u, s);
    fr_t* E2 = s.alloc<fr_t>(cols);
    eq_table_r2_dev(ctx, u, k, E2, s);
    uint32_t ln = 0;
    while ((1ull << ln) < nrows) ln++;
    if (use_tc) {
        ZK_REQUIRE(rowdot_tc_ok(nrows, cols), ZK_ERR_ARG, "shape not supported by the tensor-core row dot");
        rowdot_tc(ctx, d_M, nrows, cols, E2, static_cast<fr_t*>(d_out), 1ull << ln, ln, 1, s, use_tc == 2 ? 1 : 0);
    } else {
        ZK_LAUNCH(ctx, k_rowdot_i32<LoadPlain>, grid_for(ctx, nrows * 32, 256, 8), 256, 0, LoadPlain{d_M}, nrows, cols,
                  (const fr_t*)E2, static_cast<fr_t*>(d_out), 1ull << ln, ln, (uint64_t)1);
    }
    ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    ZK_API_END(ctx)
}

zk_status zk_diag_mul_bench(zk_ctx* ctx, const void* d_seed /* 1024 Fr */, uint32_t iters, uint32_t blocks, void* d_out) {
    ZK_API_BEGIN(ctx)
    ZK_REQUIRE(d_seed && d_out && blocks, ZK_ERR_ARG, "bad argument");
    mul_bench_dev(ctx, static_cast<const fr_t*>(d_seed), iters, blocks, static_cast<fr_t*>(d_out));
    ZK_API_END(ctx)
}

}  // extern "C"
