// shard.cu — sharded product sumcheck over G = 2^s devices (north star "sharded on its
// high variables across the 8 B200s").
//
// Rank g holds entries [g 2^L, (g+1) 2^L) of every table, L = m - s: its id is the top s bits of the
// flat index, i.e. the LAST-bound variables (D2), so every pair (2b, 2b+1) of rounds t < L is local.
// The suffix eq weight of a global pair splits as beta(w_{t+1..L-1}, b_local) * beta(w_{L..n_eq-1}, g),
// so a rank runs the single-device round kernel on its slice with its n_eq clipped to L and its K+1
// totals scaled by c_g = beta(w_{L..n_eq-1}, g) (partial-only mode).  The caller all-gathers the
// G x (K+1) partials (NCCL over NVLink / NVSwitch, or sequential virtual shards on one device) and
// zk_sc_shard_finish adds them and runs the transcript step — identically on every rank, so the
// challenges agree without a broadcast and the transcript equals the single-device one for every G.
// When the local slice gets small the folded tables are exported, all-gathered, and the remaining
// rounds run on every rank from the full tables (continuation: no second header).
#include <dlfcn.h>

#include <mutex>

#include "sumcheck.cuh"
#include "tables.cuh"

using namespace zk;

// NCCL, loaded at run time (the library loads without it; the process's libnccl.so.2 — torch's — is used
// when already loaded).  Only the five entry points the exchange needs; ABI types as in nccl.h.
namespace {
struct NcclUid {
    char internal[128];
};
struct Nccl {
    int (*get_unique_id)(NcclUid*) = nullptr;
    int (*comm_init_rank)(void**, int, NcclUid, int) = nullptr;
    int (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
    int (*comm_destroy)(void*) = nullptr;
    const char* (*error_string)(int) = nullptr;
    bool ok = false;
};
Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        n.get_unique_id = reinterpret_cast<int (*)(NcclUid*)>(dlsym(h, "ncclGetUniqueId"));
        n.comm_init_rank = reinterpret_cast<int (*)(void**, int, NcclUid, int)>(dlsym(h, "ncclCommInitRank"));
        n.all_gather = reinterpret_cast<int (*)(const void*, void*, size_t, int, void*, cudaStream_t)>(dlsym(h, "ncclAllGather"));
        n.comm_destroy = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclCommDestroy"));
        n.error_string = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
        n.ok = n.get_unique_id && n.comm_init_rank && n.all_gather && n.comm_destroy && n.error_string;
    });
    return n;
}
constexpr int NCCL_UINT8 = 1;   // ncclUint8
#define ZK_NCCL(call)                                                                                  \
    do {                                                                                               \
        const int r_ = (call);                                                                         \
        if (r_ != 0) throw ZkError{ZK_ERR_NCCL, std::string("NCCL: ") + nccl().error_string(r_)};      \
    } while (0)
}  // namespace

struct zk_sc_shard {
    zk_ctx* ctx = nullptr;
    zk_transcript* tr = nullptr;
    Scratch* s = nullptr;
    ScEngine e;
    uint32_t rank = 0, world = 1, L = 0;
    uint64_t plen = 0;
    bool done = false;
};

namespace zk {
// fold src (2 n entries) by r into dst (n entries); or plain copy when r == nullptr
__global__ void k_fold_copy(const fr_t* src, uint64_t n, const fr_t* r, fr_t* dst) {
    fr_t rr;
    if (r) rr = fr_load(r);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (r) {
            fr_t a = fr_load(&src[2 * i]), b = fr_load(&src[2 * i + 1]);
            fr_store(&dst[i], fr_add(a, fr_mul(rr, fr_sub(b, a))));
        } else {
            fr_store(&dst[i], fr_load(&src[i]));
        }
    }
}
// gathered [G][K][n] -> table k: [G * n]
__global__ void k_unshard(const fr_t* all, uint32_t G, uint32_t K, uint64_t n, uint32_t k, fr_t* out) {
    const uint64_t tot = (uint64_t)G * n;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < tot; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = i / n, j = i % n;
        fr_store(&out[i], fr_load(&all[(g * K + k) * n + j]));
    }
}
__global__ void k_pick(const fr_t* tab, uint32_t idx, fr_t* out) { fr_store(out, fr_load(&tab[idx])); }
}  // namespace zk

#define SH_BEGIN(sh)                                                                                   \
    if (!(sh)) return ZK_ERR_ARG;                                                                      \
    zk_ctx* ctx = (sh)->ctx;                                                                           \
    try {                                                                                              \
        ZK_CUDA(cudaSetDevice(ctx->device));
#define SH_END                                                                                         \
    }                                                                                                  \
    catch (const ZkError& e) {                                                                         \
        ctx->err = e.msg;                                                                              \
        return e.st;                                                                                   \
    }                                                                                                  \
    catch (const std::exception& e) {                                                                  \
        ctx->err = e.what();                                                                           \
        return ZK_ERR_INTERNAL;                                                                        \
    }                                                                                                  \
    return ZK_OK;

extern "C" {

zk_status zk_sc_shard_create(zk_ctx* ctx, zk_transcript* tr, const zk_prod_stmt* st, void* const* d_local_tables,
                             const zk_fr* claim, uint32_t rank, uint32_t world, zk_sc_shard** out) {
    if (!ctx || !out) return ZK_ERR_ARG;
    *out = nullptr;
    zk_sc_shard* sh = new zk_sc_shard();
    sh->ctx = ctx;
    try {
        ZK_CUDA(cudaSetDevice(ctx->device));
        ZK_REQUIRE(tr && st && d_local_tables, ZK_ERR_ARG, "null argument");
        const uint32_t m = st->m, n_eq = st->n_eq, K = st->n_tables;
        ZK_REQUIRE(world >= 1 && (world & (world - 1)) == 0 && rank < world, ZK_ERR_ARG, "world must be a power of two");
        uint32_t sbits = 0;
        while ((1u << sbits) < world) sbits++;
        ZK_REQUIRE(m >= 1 && m <= 40 && n_eq <= m && K >= 1 && K <= 3 && m > sbits, ZK_ERR_ARG, "bad statement / shards");
        const uint32_t L = m - sbits;
        sh->tr = tr;
        sh->rank = rank;
        sh->world = world;
        sh->L = L;
        sh->s = new Scratch(ctx);
        Scratch& s = *sh->s;
        ScEngine& e = sh->e;
        e.ctx = ctx;
        e.tr = tr;
        e.s = sh->s;
        e.m = m;
        e.n_eq = n_eq;
        e.K = K;
        fr_t* w = s.alloc<fr_t>(n_eq ? n_eq : 1);
        upload_points(ctx, st->w, n_eq, w, s);
        e.d_w = w;
        e.d_claim = s.alloc<fr_t>(1);
        if (claim) {
            upload_points(ctx, claim, 1, e.d_claim, s);
            e.claim_given = true;
        }
        sh->plen = sumcheck_proof_len(m, K);
        e.d_proof = s.alloc<uint8_t>(sh->plen);
        e.d_r = s.alloc<fr_t>(m);
        e.d_point = s.alloc<uint8_t>(32ull * m);
        e.d_finals = s.alloc<fr_t>(K);
        const fr_t* tabs[3] = {nullptr, nullptr, nullptr};
        const int32_t* i32[3] = {nullptr, nullptr, nullptr};
        for (uint32_t k = 0; k < K; k++) {
            ZK_REQUIRE(d_local_tables[k], ZK_ERR_ARG, "null table");
            if (st->i32_mask & (1u << k)) {   // embedded by round 0 (ScEngine::set_i32)
                tabs[k] = s.alloc<fr_t>(1ull << L);
                i32[k] = static_cast<const int32_t*>(d_local_tables[k]);
            } else {
                tabs[k] = static_cast<const fr_t*>(d_local_tables[k]);
            }
        }
        // rank eq factor over the high bits that the eq covers
        if (n_eq > L) {
            const uint32_t kh = n_eq - L;
            fr_t* eh = s.alloc<fr_t>(1ull << kh);
            eq_table_dev(ctx, w + L, kh, nullptr, eh, s);
            fr_t* sc = s.alloc<fr_t>(1);
            ZK_LAUNCH(ctx, k_pick, 1, 1, 0, (const fr_t*)eh, rank & ((1u << kh) - 1), sc);
            e.d_scale = sc;
        }
        e.header();
        e.setup(tabs, L, 0, n_eq < L ? n_eq : L);
        e.set_i32(i32);
    } catch (const ZkError& err) {
        ctx->err = err.msg;
        delete sh->s;
        delete sh;
        return err.st;
    }
    *out = sh;
    return ZK_OK;
}

uint32_t zk_sc_shard_rounds_done(const zk_sc_shard* sh) { return sh ? sh->e.t : 0; }
uint32_t zk_sc_shard_local_log(const zk_sc_shard* sh) { return sh ? sh->e.L - (sh->e.t - sh->e.t0) : 0; }

zk_status zk_sc_shard_partial(zk_sc_shard* sh, void* d_part) {
    SH_BEGIN(sh)
    ZK_REQUIRE(d_part && !sh->done && sh->e.t0 == 0 && sh->e.t < sh->L, ZK_ERR_ARG, "no sharded round left");
    sh->e.round(static_cast<fr_t*>(d_part));
    SH_END
}

zk_status zk_sc_shard_finish(zk_sc_shard* sh, const void* d_all) {
    SH_BEGIN(sh)
    ZK_REQUIRE(d_all && sh->e.t >= 1, ZK_ERR_ARG, "finish without partial");
    sh->e.combine(static_cast<const fr_t*>(d_all), sh->world);
    if (sh->e.t == sh->e.m) {   // the last round was sharded (m = L case cannot happen with world > 1)
        sh->e.finals();
        sh->done = true;
    }
    SH_END
}

zk_status zk_sc_shard_export(zk_sc_shard* sh, void* d_out) {
    SH_BEGIN(sh)
    ZK_REQUIRE(d_out && !sh->done && sh->e.t0 == 0, ZK_ERR_ARG, "nothing to export");
    ScEngine& e = sh->e;
    const uint64_t n = 1ull << (e.L - e.t);   // local entries after folding by r_{t-1}
    fr_t* out = static_cast<fr_t*>(d_out);
    e.materialize();
    for (uint32_t k = 0; k < e.K; k++)
        ZK_LAUNCH(ctx, k_fold_copy, grid_for(ctx, n, 256, 8), 256, 0, e.cur[k], n, e.t ? e.d_r + (e.t - 1) : nullptr,
                  out + k * n);
    SH_END
}

zk_status zk_sc_shard_adopt(zk_sc_shard* sh, const void* d_full) {
    SH_BEGIN(sh)
    ZK_REQUIRE(d_full && !sh->done && sh->e.t0 == 0, ZK_ERR_ARG, "nothing to adopt");
    ScEngine& e = sh->e;
    const uint32_t ta = e.t;
    const uint64_t n = 1ull << (e.L - ta);
    const uint32_t Lf = e.m - ta;           // log2 of the full folded tables
    const fr_t* tabs[3] = {nullptr, nullptr, nullptr};
    for (uint32_t k = 0; k < e.K; k++) {
        fr_t* full = sh->s->alloc<fr_t>(1ull << Lf);
        ZK_LAUNCH(ctx, k_unshard, grid_for(ctx, (uint64_t)sh->world * n, 256, 8), 256, 0, static_cast<const fr_t*>(d_full),
                  sh->world, e.K, n, k, full);
        tabs[k] = full;
    }
    e.d_scale = nullptr;
    e.setup(tabs, Lf, ta, e.n_eq > ta ? e.n_eq - ta : 0);
    e.run_to_end();
    sh->done = true;
    SH_END
}

zk_status zk_sc_shard_result(zk_sc_shard* sh, uint8_t* proof, uint64_t* proof_len, zk_fr* point_out, zk_fr* finals_out,
                             zk_fr* claim_out) {
    SH_BEGIN(sh)
    ZK_REQUIRE(sh->done, ZK_ERR_ARG, "sharded sumcheck not finished");
    ScEngine& e = sh->e;
    if (proof_len) {
        if (proof && *proof_len < sh->plen) {
            *proof_len = sh->plen;
            throw ZkError{ZK_ERR_ARG, "proof buffer too small"};
        }
        *proof_len = sh->plen;
    }
    if (proof) ZK_CUDA(cudaMemcpyAsync(proof, e.d_proof, sh->plen, cudaMemcpyDeviceToHost, ctx->stream));
    if (point_out) ZK_CUDA(cudaMemcpyAsync(point_out, e.d_point, 32ull * e.m, cudaMemcpyDeviceToHost, ctx->stream));
    if (finals_out)
        ZK_CUDA(cudaMemcpyAsync(finals_out, e.d_proof + 44 + 32ull * e.m * (e.K + 1), 32ull * e.K, cudaMemcpyDeviceToHost,
                                ctx->stream));
    if (claim_out) ZK_CUDA(cudaMemcpyAsync(claim_out, e.d_proof + 12, 32, cudaMemcpyDeviceToHost, ctx->stream));
    ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    SH_END
}

// ---- the exchange owned by the library (SURVEY §8(b) zk_ctx_attach_nccl; north star "allgathers partial
// round-polynomial coefficients as raw bytes via NCCL, adds them mod p on the device")
zk_status zk_nccl_unique_id(uint8_t out[128]) {
    if (!out) return ZK_ERR_ARG;
    Nccl& n = nccl();
    if (!n.ok) return ZK_ERR_NCCL;
    NcclUid id;
    if (n.get_unique_id(&id) != 0) return ZK_ERR_NCCL;
    memcpy(out, id.internal, 128);
    return ZK_OK;
}

zk_status zk_ctx_attach_nccl(zk_ctx* ctx, const uint8_t id[128], int rank, int world) {
    if (!ctx) return ZK_ERR_ARG;
    try {
        ZK_CUDA(cudaSetDevice(ctx->device));
        ZK_REQUIRE(id && world >= 1 && rank >= 0 && rank < world && (world & (world - 1)) == 0, ZK_ERR_ARG,
                   "need 0 <= rank < world, world a power of two");
        Nccl& n = nccl();
        ZK_REQUIRE(n.ok, ZK_ERR_NCCL, "libnccl.so.2 not found");
        if (ctx->nccl_comm) ZK_NCCL(n.comm_destroy(ctx->nccl_comm));
        ctx->nccl_comm = nullptr;
        NcclUid uid;
        memcpy(uid.internal, id, 128);
        void* comm = nullptr;
        ZK_NCCL(n.comm_init_rank(&comm, world, uid, rank));
        ctx->nccl_comm = comm;
        ctx->nccl_rank = rank;
        ctx->nccl_world = world;
    } catch (const ZkError& e) {
        ctx->err = e.msg;
        return e.st;
    }
    return ZK_OK;
}

zk_status zk_ctx_detach_nccl(zk_ctx* ctx) {
    if (!ctx) return ZK_ERR_ARG;
    if (ctx->nccl_comm) {
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        nccl().comm_destroy(ctx->nccl_comm);
        ctx->nccl_comm = nullptr;
    }
    return ZK_OK;
}

// Every remaining round of a sharded statement with the exchange inside the library: per round the
// K+1 partials (32-byte elements) are all-gathered as raw bytes (ncclUint8) on the context stream and
// added mod p on the device with the transcript step; below 2^switch_log local entries the folded
// tables are all-gathered and every rank finishes alone.  No host synchronisation, no per-round host
// logic beyond the round counter; collect the proof with zk_sc_shard_result.
zk_status zk_sc_shard_prove_nccl(zk_sc_shard* sh, uint32_t switch_log) {
    SH_BEGIN(sh)
    ZK_REQUIRE(ctx->nccl_comm && ctx->nccl_world == (int)sh->world && ctx->nccl_rank == (int)sh->rank, ZK_ERR_ARG,
               "context not attached to an NCCL communicator of this shard's rank and world");
    ScEngine& e = sh->e;
    Nccl& n = nccl();
    const uint64_t pbytes = 32ull * (e.K + 1);
    fr_t* part = sh->s->alloc<fr_t>(e.K + 1);
    fr_t* all = sh->s->alloc<fr_t>((uint64_t)sh->world * (e.K + 1));
    while (!sh->done && e.t0 == 0 && e.t < sh->L && (e.L - e.t) > switch_log) {
        e.round(part);
        ZK_NCCL(n.all_gather(part, all, pbytes, NCCL_UINT8, ctx->nccl_comm, ctx->stream));
        e.combine(all, sh->world);
        if (e.t == e.m) {
            e.finals();
            sh->done = true;
        }
    }
    if (!sh->done) {
        const uint64_t nloc = 1ull << (e.L - e.t);
        fr_t* loc = sh->s->alloc<fr_t>(e.K * nloc);
        fr_t* full = sh->s->alloc<fr_t>((uint64_t)sh->world * e.K * nloc);
        e.materialize();
        for (uint32_t k = 0; k < e.K; k++)
            ZK_LAUNCH(ctx, k_fold_copy, grid_for(ctx, nloc, 256, 8), 256, 0, e.cur[k], nloc,
                      e.t ? e.d_r + (e.t - 1) : nullptr, loc + k * nloc);
        ZK_NCCL(n.all_gather(loc, full, 32ull * e.K * nloc, NCCL_UINT8, ctx->nccl_comm, ctx->stream));
        const uint32_t ta = e.t;
        const uint32_t Lf = e.m - ta;
        const fr_t* tabs[3] = {nullptr, nullptr, nullptr};
        for (uint32_t k = 0; k < e.K; k++) {
            fr_t* t = sh->s->alloc<fr_t>(1ull << Lf);
            ZK_LAUNCH(ctx, k_unshard, grid_for(ctx, (uint64_t)sh->world * nloc, 256, 8), 256, 0, (const fr_t*)full,
                      sh->world, e.K, nloc, k, t);
            tabs[k] = t;
        }
        e.d_scale = nullptr;
        e.setup(tabs, Lf, ta, e.n_eq > ta ? e.n_eq - ta : 0);
        e.run_to_end();
        sh->done = true;
    }
    SH_END
}

void zk_sc_shard_free(zk_sc_shard* sh) {
    if (!sh) return;
    cudaSetDevice(sh->ctx->device);
    delete sh->s;   // stream-ordered frees
    cudaStreamSynchronize(sh->ctx->stream);
    delete sh;
}

}  // extern "C"
