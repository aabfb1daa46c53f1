// transcript.cu — Fiat-Shamir transcript kernels and host wrappers (D3; row a6).
#include "common.cuh"

namespace zk {

__global__ void k_tr_init(uint8_t* st, Bytes256 seed) { tr_init(st, seed.b); }

__global__ void k_tr_absorb(uint8_t* st, Tag32 tag, Bytes256 msg) {
    if (threadIdx.x == 0 && blockIdx.x == 0) tr_absorb(st, tag.s, msg.b, msg.len);
}

__global__ void k_tr_absorb_dev(uint8_t* st, Tag32 tag, const uint8_t* msg, uint64_t len) {
    if (threadIdx.x == 0 && blockIdx.x == 0) tr_absorb(st, tag.s, msg, len);
}

__global__ void k_tr_absorb_frs(uint8_t* st, Tag32 tag, const fr_t* v, uint32_t n, uint8_t* copy_out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        Sha256 s;
        tr_absorb_begin(s, st, tag.s, 32ull * n);
        for (uint32_t i = 0; i < n; i++) {
            uint8_t b[32];
            fr_to_bytes(fr_load(&v[i]), b);
            s.update(b, 32);
            if (copy_out)
                for (int k = 0; k < 32; k++) copy_out[32 * i + k] = b[k];
        }
        s.final(st);
    }
}

// Squeeze x = LE512(SHA256(st||0) || SHA256(st||1)) mod p for one challenge state.
__device__ fr_t squeeze_from_state(const uint8_t* st) {
    Sha256 s;
    uint8_t h[64];
    for (int k = 0; k < 2; k++) {
        s.init();
        s.update(st, 32);
        s.update_byte((uint8_t)k);
        s.final(h + 32 * k);
    }
    fr_t lo, hi;
    for (int i = 0; i < 8; i++) {
        lo.v[i] = (uint32_t)h[4 * i] | ((uint32_t)h[4 * i + 1] << 8) | ((uint32_t)h[4 * i + 2] << 16) |
                  ((uint32_t)h[4 * i + 3] << 24);
        hi.v[i] = (uint32_t)h[32 + 4 * i] | ((uint32_t)h[33 + 4 * i] << 8) | ((uint32_t)h[34 + 4 * i] << 16) |
                  ((uint32_t)h[35 + 4 * i] << 24);
    }
    return fr_add(fr_mul(ZK_R2, lo), fr_mul(ZK_R3, hi));
}

// blockDim.x >= 1; n <= 256 per launch (the host splits larger requests)
__global__ void k_tr_challenges(uint8_t* st, Tag32 tag, uint32_t n, fr_t* out_mont, uint8_t* out_canon) {
    __shared__ uint8_t states[256][32];
    if (threadIdx.x == 0) {
        uint32_t tl = zk_strlen(tag.s);
        for (uint32_t i = 0; i < n; i++) {
            Sha256 s;
            s.init();
            s.update(st, 32);
            s.update_byte(0x02);
            s.update_byte((uint8_t)tl);
            s.update((const uint8_t*)tag.s, tl);
            s.final(st);
            for (int k = 0; k < 32; k++) states[i][k] = st[k];
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        fr_t x = squeeze_from_state(states[i]);
        if (out_mont) fr_store(&out_mont[i], x);
        if (out_canon) fr_to_bytes(x, out_canon + 32 * i);
    }
}

void tr_absorb_host(zk_transcript* tr, const char* tag, const void* msg, size_t len) {
    zk_ctx* ctx = tr->ctx;
    if (len <= 256) {
        ZK_LAUNCH(ctx, k_tr_absorb, 1, 32, 0, tr->d_st, make_tag(tag), make_bytes(msg, len));
    } else {
        Scratch s(ctx);
        uint8_t* d = s.alloc<uint8_t>(len);
        ZK_CUDA(cudaMemcpyAsync(d, msg, len, cudaMemcpyHostToDevice, ctx->stream));
        ZK_LAUNCH(ctx, k_tr_absorb_dev, 1, 32, 0, tr->d_st, make_tag(tag), d, (uint64_t)len);
        ZK_CUDA(cudaStreamSynchronize(ctx->stream));   // msg is a pageable host buffer
    }
}

void tr_challenges_dev(zk_transcript* tr, const char* tag, uint32_t n, fr_t* d_out_mont, uint8_t* d_out_canon) {
    zk_ctx* ctx = tr->ctx;
    Tag32 t = make_tag(tag);
    for (uint32_t off = 0; off < n; off += 256) {
        uint32_t c = n - off < 256 ? n - off : 256;
        ZK_LAUNCH(ctx, k_tr_challenges, 1, 256, 0, tr->d_st, t, c, d_out_mont ? d_out_mont + off : nullptr,
                  d_out_canon ? d_out_canon + 32 * (size_t)off : nullptr);
    }
}

void tr_init_dev(zk_transcript* tr, const uint8_t seed[32]) {
    ZK_LAUNCH(tr->ctx, k_tr_init, 1, 1, 0, tr->d_st, make_bytes(seed, 32));
}

}  // namespace zk
