// transcript.cu — Fiat-Shamir transcript kernels and host wrappers (D3; row a6).
// Every kernel here is launched with one warp (or a block whose warp 0 runs the transcript).
#include <cstring>

#include "common.cuh"

namespace zk {

__global__ void k_tr_init(uint8_t* st, Bytes256 seed) {
    __shared__ uint32_t buf[32];
    if (threadIdx.x == 0) {
        uint8_t* b = reinterpret_cast<uint8_t*>(buf);
        const char* lbl = "zkdl-b200/v1/init";
        uint32_t n = zk_strlen(lbl);
        for (uint32_t i = 0; i < n; i++) b[i] = (uint8_t)lbl[i];
        for (int i = 0; i < 32; i++) b[n + i] = seed.b[i];
        uint32_t d[8];
        hash_buf(b, n + 32, d);
        st_words_to_bytes(d, st);
    }
}

// copy_out (nullable): the message bytes are also written there (proof headers without a host copy)
__global__ void k_tr_absorb(uint8_t* st, Tag32 tag, Bytes256 msg, uint8_t* copy_out) {
    __shared__ FsScratch s;
    if (copy_out)
        for (uint32_t i = threadIdx.x; i < msg.len; i += blockDim.x) copy_out[i] = msg.b[i];
    fs_begin(s, st);
    fs_absorb_bytes(s, tag.s, msg.b, msg.len);
    fs_end(s, st);
}

// messages from device memory: up to 256 bytes through the warp-assembled path (fs_absorb_bytes: the 32
// lanes build the blocks in shared memory, lane 0 compresses); longer ones streamed by lane 0
__global__ void k_tr_absorb_dev(uint8_t* st, Tag32 tag, const uint8_t* msg, uint64_t len) {
    if (len <= 256) {
        __shared__ FsScratch s;
        __shared__ uint8_t m[256];
        for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) m[i] = msg[i];
        __syncwarp();
        fs_begin(s, st);
        fs_absorb_bytes(s, tag.s, m, (uint32_t)len);
        fs_end(s, st);
        return;
    }
    if (threadIdx.x != 0) return;
    __shared__ uint32_t buf[32];
    uint8_t* b = reinterpret_cast<uint8_t*>(buf);
    uint32_t h[8];
    hash_init(h);
    // header
    uint8_t hdr[80];
    for (int i = 0; i < 32; i++) hdr[i] = st[i];
    uint32_t tl = zk_strlen(tag.s);
    hdr[32] = 0x01;
    hdr[33] = (uint8_t)tl;
    for (uint32_t i = 0; i < tl; i++) hdr[34 + i] = (uint8_t)tag.s[i];
    for (int i = 0; i < 8; i++) hdr[34 + tl + i] = (uint8_t)(len >> (56 - 8 * i));
    const uint64_t hl = 42 + tl, total = hl + len;
    const uint64_t nb = total == 0 ? 1 : (total + 63) / 64;
    for (uint64_t blk = 0; blk < nb; blk++) {
        const uint64_t off = 64 * blk;
        for (int i = 0; i < 64; i++) {
            const uint64_t p = off + i;
            b[i] = p < hl ? hdr[p] : p < total ? msg[p - hl] : 0;
        }
        hash_compress(h, buf, (uint32_t)(total < off + 64 ? total : off + 64), blk + 1 == nb);
    }
    st_words_to_bytes(h, st);
}

// Fork (D3d): the parent draws challenge `tag`; the child's initial state is
// H("zkdl-b200/v1/init" || canonical bytes of that challenge), i.e. a transcript seeded with it.
__global__ void k_tr_fork(uint8_t* st, Tag32 tag, uint8_t* child_st) {
    __shared__ FsScratch s;
    __shared__ uint32_t buf[32];
    fs_begin(s, st);
    fs_challenge(s, tag.s);
    if (threadIdx.x == 0) {
        uint8_t* b = reinterpret_cast<uint8_t*>(buf);
        const char* lbl = "zkdl-b200/v1/init";
        const uint32_t n = zk_strlen(lbl);
        for (uint32_t i = 0; i < n; i++) b[i] = (uint8_t)lbl[i];
        fr_canon_to_bytes(s.rc, b + n);
        uint32_t d[8];
        hash_buf(b, n + 32, d);
        st_words_to_bytes(d, child_st);
    }
    fs_end(s, st);
}

// n <= 8 field elements from device memory (Montgomery)
__global__ void k_tr_absorb_frs(uint8_t* st, Tag32 tag, const fr_t* v, uint32_t n, uint8_t* copy_out) {
    __shared__ FsScratch s;
    const int lane = threadIdx.x & 31;
    fs_begin(s, st);
    fr_t mine = lane < (int)n ? fr_load(&v[lane]) : fr_zero();
    fs_absorb_frs(s, tag.s, mine, (int)n, copy_out);
    fs_end(s, st);
}

// n challenges with one tag (D3: st_{i+1} = H(st_i || 0x02 || u8(|tag|) || tag), x_i = LE512(H(st_{i+1} || 0) ||
// H(st_{i+1} || 1)) mod p).  Thread 0 advances the state chain word-wise (the block's tail after the state
// is the same for every step: built once), then thread j < 2n computes squeeze half j & 1 of challenge
// j / 2, and thread i < n converts.  blockDim.x >= max(32, 2n); n <= 256 per launch.
// Up to TRM_MAX challenge vectors (tags) in one launch, drawn in order (the same chain as one launch per tag).
constexpr int TRM_MAX = 4;
struct TrMulti {
    Tag32 tag[TRM_MAX];
    uint32_t n[TRM_MAX];
    fr_t* out_mont[TRM_MAX];
    uint8_t* out_canon[TRM_MAX];
    uint32_t ntag;
};
__global__ void k_tr_challenges_multi(uint8_t* st, TrMulti a) {
    __shared__ uint32_t states[256][8];
    __shared__ fr_t half[256][2];
    __shared__ uint32_t m[16];   // the chain's message block (shared memory: the compression reads it in place)
    uint32_t total = 0;
    for (uint32_t t = 0; t < a.ntag; t++) total += a.n[t];
    if (threadIdx.x == 0) {
        uint32_t cur[8];
#pragma unroll
        for (int k = 0; k < 8; k++)
            cur[k] = (uint32_t)st[4 * k] | ((uint32_t)st[4 * k + 1] << 8) | ((uint32_t)st[4 * k + 2] << 16) |
                     ((uint32_t)st[4 * k + 3] << 24);
        uint32_t idx = 0;
        for (uint32_t t = 0; t < a.ntag; t++) {
            const uint32_t tl = zk_strlen(a.tag[t].s);
#pragma unroll
            for (int k = 8; k < 16; k++) m[k] = 0;
            // bytes 32.. of the block: 0x02, |tag|, tag (|tag| <= 30)
            uint8_t* tb = reinterpret_cast<uint8_t*>(m + 8);
            tb[0] = 0x02;
            tb[1] = (uint8_t)tl;
            for (uint32_t k = 0; k < tl; k++) tb[2 + k] = (uint8_t)a.tag[t].s[k];
            for (uint32_t i = 0; i < a.n[t]; i++, idx++) {
#pragma unroll
                for (int k = 0; k < 8; k++) m[k] = cur[k];
                hash_init(cur);
                hash_compress(cur, m, 34 + tl, true);
#pragma unroll
                for (int k = 0; k < 8; k++) states[idx][k] = cur[k];
            }
        }
        st_words_to_bytes(cur, st);
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < 2 * total; j += blockDim.x) {   // one squeeze compression: H(st_i || k)
        const uint32_t i = j >> 1, k = j & 1;
        uint32_t q[16], d[8];
#pragma unroll
        for (int w = 0; w < 8; w++) q[w] = states[i][w];
        q[8] = k;
#pragma unroll
        for (int w = 9; w < 16; w++) q[w] = 0;
        hash_init(d);
        hash_compress(d, q, 33, true);
        fr_t x;
#pragma unroll
        for (int w = 0; w < 8; w++) x.v[w] = d[w];   // little-endian digest words = limbs
        half[i][k] = x;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) {
        uint32_t t = 0, o = i;
        while (o >= a.n[t]) o -= a.n[t++];
        const fr_t lo = half[i][0], hi = half[i][1];
        if (a.out_mont[t]) fr_store(&a.out_mont[t][o], fr_add(fr_mul(ZK_R2, lo), fr_mul(ZK_R3, hi)));
        if (a.out_canon[t])
            fr_canon_to_bytes(fr_add(fr_reduce_once(fr_reduce_once(lo)), fr_mul(ZK_R2, hi)), a.out_canon[t] + 32 * o);
    }
}

// n challenges with one tag (D3: st_{i+1} = H(st_i || 0x02 || u8(|tag|) || tag), x_i = LE512(H(st_{i+1} || 0) ||
// H(st_{i+1} || 1)) mod p).  Thread 0 advances the state chain word-wise (the block's tail after the state
// is the same for every step: built once), then thread j < 2n computes squeeze half j & 1 of challenge
// j / 2, and thread i < n converts.  blockDim.x >= max(32, 2n); n <= 256 per launch.
__global__ void k_tr_challenges(uint8_t* st, Tag32 tag, uint32_t n, fr_t* out_mont, uint8_t* out_canon) {
    __shared__ uint32_t states[256][8];
    __shared__ fr_t half[256][2];
    __shared__ uint32_t m[16];   // the chain's message block (shared memory: the compression reads it in place)
    if (threadIdx.x == 0) {
        const uint32_t tl = zk_strlen(tag.s);
#pragma unroll
        for (int k = 8; k < 16; k++) m[k] = 0;
        // bytes 32.. of the block: 0x02, |tag|, tag (|tag| <= 30)
        uint8_t* tb = reinterpret_cast<uint8_t*>(m + 8);
        tb[0] = 0x02;
        tb[1] = (uint8_t)tl;
        for (uint32_t k = 0; k < tl; k++) tb[2 + k] = (uint8_t)tag.s[k];
        uint32_t cur[8];
#pragma unroll
        for (int k = 0; k < 8; k++)
            cur[k] = (uint32_t)st[4 * k] | ((uint32_t)st[4 * k + 1] << 8) | ((uint32_t)st[4 * k + 2] << 16) |
                     ((uint32_t)st[4 * k + 3] << 24);
        for (uint32_t i = 0; i < n; i++) {
#pragma unroll
            for (int k = 0; k < 8; k++) m[k] = cur[k];
            hash_init(cur);
            hash_compress(cur, m, 34 + tl, true);
#pragma unroll
            for (int k = 0; k < 8; k++) states[i][k] = cur[k];
        }
        st_words_to_bytes(cur, st);
    }
    __syncthreads();
    if (threadIdx.x < 2 * n) {   // one squeeze compression per thread: H(st_i || k), 33 bytes
        const uint32_t i = threadIdx.x >> 1, k = threadIdx.x & 1;
        uint32_t q[16], d[8];
#pragma unroll
        for (int w = 0; w < 8; w++) q[w] = states[i][w];
        q[8] = k;
#pragma unroll
        for (int w = 9; w < 16; w++) q[w] = 0;
        hash_init(d);
        hash_compress(d, q, 33, true);
        fr_t x;
#pragma unroll
        for (int w = 0; w < 8; w++) x.v[w] = d[w];   // little-endian digest words = limbs
        half[i][k] = x;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const fr_t lo = half[i][0], hi = half[i][1];
        if (out_mont) fr_store(&out_mont[i], fr_add(fr_mul(ZK_R2, lo), fr_mul(ZK_R3, hi)));
        if (out_canon) fr_canon_to_bytes(fr_add(fr_reduce_once(fr_reduce_once(lo)), fr_mul(ZK_R2, hi)), out_canon + 32 * i);
    }
}

void tr_absorb_host(zk_transcript* tr, const char* tag, const void* msg, size_t len, uint8_t* d_copy) {
    zk_ctx* ctx = tr->ctx;
    if (len <= 256) {
        ZK_LAUNCH(ctx, k_tr_absorb, 1, 32, 0, tr->d_st, make_tag(tag), make_bytes(msg, len), d_copy);
    } else {
        ZK_REQUIRE(d_copy == nullptr, ZK_ERR_INTERNAL, "copy-out only for short messages");
        Scratch s(ctx);
        uint8_t* d = s.alloc<uint8_t>(len);
        ZK_CUDA(cudaMemcpyAsync(d, msg, len, cudaMemcpyHostToDevice, ctx->stream));
        ZK_LAUNCH(ctx, k_tr_absorb_dev, 1, 32, 0, tr->d_st, make_tag(tag), d, (uint64_t)len);
        ZK_CUDA(cudaStreamSynchronize(ctx->stream));   // msg is a pageable host buffer
    }
}

void tr_challenges_multi_dev(zk_transcript* tr, uint32_t k, const char* const* tags, const uint32_t* ns,
                             fr_t* const* d_out_mont, uint8_t* const* d_out_canon) {
    ZK_REQUIRE(k >= 1 && k <= (uint32_t)TRM_MAX, ZK_ERR_ARG, "1..4 challenge vectors per launch");
    TrMulti a;
    memset(&a, 0, sizeof a);
    uint32_t total = 0;
    for (uint32_t t = 0; t < k; t++) {
        ZK_REQUIRE(strlen(tags[t]) <= 30, ZK_ERR_ARG, "challenge tag longer than 30 bytes (one-block chain step)");
        a.tag[t] = make_tag(tags[t]);
        a.n[t] = ns[t];
        a.out_mont[t] = d_out_mont[t];
        a.out_canon[t] = d_out_canon ? d_out_canon[t] : nullptr;
        total += ns[t];
    }
    a.ntag = k;
    if (total > 256) {   // one launch per vector
        for (uint32_t t = 0; t < k; t++) tr_challenges_dev(tr, tags[t], ns[t], d_out_mont[t], a.out_canon[t]);
        return;
    }
    ZK_LAUNCH(tr->ctx, k_tr_challenges_multi, 1, 256, 0, tr->d_st, a);
}

void tr_challenges_dev(zk_transcript* tr, const char* tag, uint32_t n, fr_t* d_out_mont, uint8_t* d_out_canon) {
    zk_ctx* ctx = tr->ctx;
    ZK_REQUIRE(strlen(tag) <= 30, ZK_ERR_ARG, "challenge tag longer than 30 bytes (one-block chain step)");
    Tag32 t = make_tag(tag);
    for (uint32_t off = 0; off < n; off += 256) {
        uint32_t c = n - off < 256 ? n - off : 256;
        uint32_t threads = (2 * c + 31) / 32 * 32;
        ZK_LAUNCH(ctx, k_tr_challenges, 1, threads, 0, tr->d_st, t, c, d_out_mont ? d_out_mont + off : nullptr,
                  d_out_canon ? d_out_canon + 32 * (size_t)off : nullptr);
    }
}

void tr_init_dev(zk_transcript* tr, const uint8_t seed[32]) {
    ZK_LAUNCH(tr->ctx, k_tr_init, 1, 32, 0, tr->d_st, make_bytes(seed, 32));
}

void tr_fork_dev(zk_transcript* parent, const char* tag, uint8_t* d_child_st) {
    ZK_LAUNCH(parent->ctx, k_tr_fork, 1, 32, 0, parent->d_st, make_tag(tag), d_child_st);
}

void tr_absorb_state_dev(zk_transcript* tr, const char* tag, const uint8_t* d_other_st) {
    ZK_LAUNCH(tr->ctx, k_tr_absorb_dev, 1, 32, 0, tr->d_st, make_tag(tag), d_other_st, (uint64_t)32);
}

}  // namespace zk

namespace zk {
// Diagnostics: latency of the per-round transcript step (absorb K+1 = 3 elements, squeeze one challenge),
// and of the out-of-line field multiply, on one warp.  mode 0: full step, 1: hash (BLAKE2s) compressions only,
// 2: fr_mul_cold chain.
__global__ void k_diag_fs(uint8_t* st, uint32_t n, int mode, fr_t* out) {
    __shared__ FsScratch fs;
    fs_begin(fs, st);
    const int lane = threadIdx.x & 31;
    fr_t v = fr_one();
    if (mode == 0) {
        for (uint32_t i = 0; i < n; i++) {
            fs_absorb_frs(fs, "sc/msg", v, 3, nullptr);
            v = fs_challenge(fs, "sc/r");
        }
    } else if (mode == 1) {
        if (lane == 0) {
            uint32_t h[8] = {1, 2, 3, 4, 5, 6, 7, 8};
            for (uint32_t i = 0; i < n; i++) hash_compress(h, fs.buf[0], 64, false);
            v.v[0] = h[0];
        }
    } else {
        if (lane == 0)
            for (uint32_t i = 0; i < n; i++) v = fr_mul_cold(v, ZK_R2);
    }
    if (lane == 0) fr_store(out, v);
    fs_end(fs, st);
}
}  // namespace zk

extern "C" zk_status zk_diag_fs_bench(zk_transcript* tr, uint32_t n, int mode, void* d_out) {
    if (!tr) return ZK_ERR_ARG;
    zk_ctx* ctx = tr->ctx;
    try {
        ZK_LAUNCH(ctx, zk::k_diag_fs, 1, 32, 0, tr->d_st, n, mode, static_cast<zk::fr_t*>(d_out));
    } catch (const zk::ZkError& e) {
        ctx->err = e.msg;
        return e.st;
    }
    return ZK_OK;
}
