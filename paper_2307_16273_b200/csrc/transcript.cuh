// transcript.cuh — device-resident Fiat-Shamir transcript (D3).
//
// The paper's protocols are interactive ("chosen by the verifier"); the
// challenges here come from a hash transcript (H = BLAKE2s-256, RFC 7693) whose 32-byte state lives
// in device memory so a whole sumcheck runs without a host round trip:
//   st0            = H("zkdl-b200/v1/init" || seed32)
//   absorb(tag, m) : st = H(st || 0x01 || u8(|tag|) || tag || u64be(|m|) || m)
//   challenge(tag) : st = H(st || 0x02 || u8(|tag|) || tag)
//                    x  = LE512(H(st || 0x00) || H(st || 0x01)) mod p
//
// Latency matters (one transcript step per sumcheck round), so the step runs on one WARP of the
// finalizing block: messages are assembled in shared memory and hashed word-wise with the round
// function fully unrolled in registers; the field elements of a message are canonicalised by
// parallel lanes; the two squeeze hashes and the four half-reductions of the 512-bit challenge
// run on separate lanes.  x = lo + hi 2^256:  mont(x) = mont_mul(R^2, lo) + mont_mul(R^3, hi),
// canonical(x) = (lo mod p) + mont_mul(R^2, hi).
// BLAKE2s rather than SHA-256: a single-warp hash is bound by the ALU pipe (2 cycles per operation
// per SMSP); BLAKE2s needs ~960 add/xor/rotate operations per 64-byte block against ~1900 for SHA-256
// (no message schedule), which halves the serial transcript latency of every round.
#pragma once
#include "fr.cuh"

namespace zk {

__device__ __forceinline__ uint32_t ror32(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

struct Hs8 {
    uint32_t h[8];
};

// BLAKE2s G; the message-word schedule (sigma) is resolved at compile time by the full unroll.
#define ZK_B2_G(a, b, c, d, x, y)                                                                      \
    do {                                                                                               \
        a += b + (x);                                                                                  \
        d = ror32(d ^ a, 16);                                                                          \
        c += d;                                                                                        \
        b = ror32(b ^ c, 12);                                                                          \
        a += b + (y);                                                                                  \
        d = ror32(d ^ a, 8);                                                                           \
        c += d;                                                                                        \
        b = ror32(b ^ c, 7);                                                                           \
    } while (0)

// One compression F(h, m, t, f) of a 64-byte block (16 little-endian words): t = bytes hashed so far
// including this block (messages here are < 2^32 bytes), last = final-block flag.  One out-of-line
// copy (~1K instructions) shared by every call site.
static __device__ __noinline__ Hs8 blake2s_compress_s(Hs8 s, const uint32_t* blk, uint32_t t, uint32_t last) {
    static constexpr uint8_t SIG[10][16] = {
        {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
        {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
        {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
        {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
        {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0}};
    uint32_t m[16];
#pragma unroll
    for (int i = 0; i < 16; i++) m[i] = blk[i];
    uint32_t v[16] = {s.h[0], s.h[1], s.h[2], s.h[3], s.h[4], s.h[5], s.h[6], s.h[7],
                      0x6A09E667u, 0xBB67AE85u, 0x3C6EF372u, 0xA54FF53Au, 0x510E527Fu ^ t, 0x9B05688Cu,
                      last ? ~0x1F83D9ABu : 0x1F83D9ABu, 0x5BE0CD19u};
#pragma unroll
    for (int r = 0; r < 10; r++) {
        ZK_B2_G(v[0], v[4], v[8], v[12], m[SIG[r][0]], m[SIG[r][1]]);
        ZK_B2_G(v[1], v[5], v[9], v[13], m[SIG[r][2]], m[SIG[r][3]]);
        ZK_B2_G(v[2], v[6], v[10], v[14], m[SIG[r][4]], m[SIG[r][5]]);
        ZK_B2_G(v[3], v[7], v[11], v[15], m[SIG[r][6]], m[SIG[r][7]]);
        ZK_B2_G(v[0], v[5], v[10], v[15], m[SIG[r][8]], m[SIG[r][9]]);
        ZK_B2_G(v[1], v[6], v[11], v[12], m[SIG[r][10]], m[SIG[r][11]]);
        ZK_B2_G(v[2], v[7], v[8], v[13], m[SIG[r][12]], m[SIG[r][13]]);
        ZK_B2_G(v[3], v[4], v[9], v[14], m[SIG[r][14]], m[SIG[r][15]]);
    }
#pragma unroll
    for (int i = 0; i < 8; i++) s.h[i] ^= v[i] ^ v[i + 8];
    return s;
}
__device__ __forceinline__ void hash_init(uint32_t h[8]) {
    h[0] = 0x6A09E667u ^ 0x01010020u;   // parameter block: 32-byte digest, unkeyed, fanout 1, depth 1
    h[1] = 0xBB67AE85u; h[2] = 0x3C6EF372u; h[3] = 0xA54FF53Au;
    h[4] = 0x510E527Fu; h[5] = 0x9B05688Cu; h[6] = 0x1F83D9ABu; h[7] = 0x5BE0CD19u;
}
__device__ __forceinline__ void hash_compress(uint32_t h[8], const uint32_t* blk, uint32_t t, bool last) {
    Hs8 s;
#pragma unroll
    for (int i = 0; i < 8; i++) s.h[i] = h[i];
    s = blake2s_compress_s(s, blk, t, last ? 1u : 0u);
#pragma unroll
    for (int i = 0; i < 8; i++) h[i] = s.h[i];
}
// blocks of an n-byte message: the final (possibly partial, zero-padded) block carries the flag; the
// empty message is one zero block
__device__ __forceinline__ uint32_t hash_nblocks(uint32_t n) { return n == 0 ? 1u : (n + 63) / 64; }

// H of n bytes held in a 4-byte-aligned buffer with capacity >= 64 * hash_nblocks(n); the tail of the
// last block is zeroed in place.  out: digest words (little-endian: state byte 4i + k = byte k of out[i]).
__device__ inline void hash_buf(uint8_t* buf, uint32_t n, uint32_t out[8]) {
    const uint32_t nb = hash_nblocks(n);
    for (uint32_t i = n; i < 64 * nb; i++) buf[i] = 0;
    uint32_t h[8];
    hash_init(h);
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(buf);
    for (uint32_t blk = 0; blk < nb; blk++) hash_compress(h, wp + 16 * blk, min(64 * (blk + 1), n), blk + 1 == nb);
#pragma unroll
    for (int i = 0; i < 8; i++) out[i] = h[i];
}

__device__ __forceinline__ uint32_t zk_strlen(const char* s) {
    uint32_t n = 0;
    while (s[n]) n++;
    return n;
}

// digest words -> the 32 state bytes (little-endian words)
__device__ __forceinline__ void st_words_to_bytes(const uint32_t w[8], uint8_t* out) {
    for (int i = 0; i < 8; i++) {
        out[4 * i] = (uint8_t)w[i];
        out[4 * i + 1] = (uint8_t)(w[i] >> 8);
        out[4 * i + 2] = (uint8_t)(w[i] >> 16);
        out[4 * i + 3] = (uint8_t)(w[i] >> 24);
    }
}

// Montgomery -> canonical integer in [0, p): one Montgomery reduction of the 256-bit value (no product;
// ~3x shorter dependency chain than fr_to_canonical_cold's product by 1)
__device__ inline fr_t fr_from_mont_fast(const fr_t& a) {
    const uint32_t w[10] = {a.v[0], a.v[1], a.v[2], a.v[3], a.v[4], a.v[5], a.v[6], a.v[7], 0u, 0u};
    return fr_redc_wide(w);
}
// Canonical 32-byte little-endian encoding of a Montgomery element.
__device__ inline void fr_to_bytes(const fr_t& a, uint8_t* out) {
    fr_t c = fr_from_mont_fast(a);
    for (int i = 0; i < 8; i++) {
        out[4 * i] = (uint8_t)c.v[i];
        out[4 * i + 1] = (uint8_t)(c.v[i] >> 8);
        out[4 * i + 2] = (uint8_t)(c.v[i] >> 16);
        out[4 * i + 3] = (uint8_t)(c.v[i] >> 24);
    }
}
__device__ inline void fr_canon_to_bytes(const fr_t& c, uint8_t* out) {
    for (int i = 0; i < 8; i++) {
        out[4 * i] = (uint8_t)c.v[i];
        out[4 * i + 1] = (uint8_t)(c.v[i] >> 8);
        out[4 * i + 2] = (uint8_t)(c.v[i] >> 16);
        out[4 * i + 3] = (uint8_t)(c.v[i] >> 24);
    }
}

// ---------------------------------------------------------------- warp-cooperative transcript steps
// The steps are out-of-line (one copy per kernel image): they run once per round on the critical path, and
// the inlined copies made the persistent round kernels large enough to re-fetch their code from L2 every
// round (k_sc_all: absorb + challenge 9.7 + 7.0 us in the kernel against 4.1 + 3.4 us alone).
// Shared scratch of one finalizing warp.
struct FsScratch {
    uint32_t buf[2][96];   // two 384-byte message buffers (header <= 73 B + payload <= 256 B, whole blocks)
    uint8_t st[32];        // current state bytes
    uint8_t pay[256];      // payload (canonical field elements) of an absorb
    fr_t part[4];
    fr_t half[2];
    fr_t r;
    fr_t rc;               // canonical r
};

// lanes copy the global state in / out
__device__ __forceinline__ void fs_begin(FsScratch& s, const uint8_t* st_g) {
    const int lane = threadIdx.x & 31;
    s.st[lane] = st_g[lane];
    __syncwarp();
}
__device__ __forceinline__ void fs_end(FsScratch& s, uint8_t* st_g) {
    __syncwarp();
    const int lane = threadIdx.x & 31;
    st_g[lane] = s.st[lane];
    __syncwarp();
}

// The 32 lanes assemble the message  st || dom || u8(|tag|) || tag || [u64be(plen)] || payload  (zero
// tail to a whole block) into s.buf[which] (each lane a strided subset of the bytes), then lane `hasher`
// compresses it and writes the digest to `out` (state bytes).  Every lane of the warp must call.
__device__ inline void fs_hash_msg(FsScratch& s, int which, uint8_t dom, const char* tag, uint32_t tl, bool with_len,
                                   const uint8_t* pay, uint32_t plen, int hasher, uint8_t* out) {
    const int lane = threadIdx.x & 31;
    uint8_t* b = reinterpret_cast<uint8_t*>(s.buf[which]);
    const uint32_t hl = 34 + tl + (with_len ? 8 : 0);
    const uint32_t total = hl + plen;
    const uint32_t nb = hash_nblocks(total);
    for (uint32_t p = lane; p < 64 * nb; p += 32) {
        uint8_t v;
        if (p < 32) v = s.st[p];
        else if (p == 32) v = dom;
        else if (p == 33) v = (uint8_t)tl;
        else if (p < 34 + tl) v = (uint8_t)tag[p - 34];
        else if (p < hl) v = (uint8_t)((uint64_t)plen >> (56 - 8 * (p - 34 - tl)));
        else if (p < total) v = pay[p - hl];
        else v = 0;
        b[p] = v;
    }
    __syncwarp();
    if (lane == hasher) {
        uint32_t h[8];
        hash_init(h);
        for (uint32_t blk = 0; blk < nb; blk++) hash_compress(h, s.buf[which] + 16 * blk, min(64 * (blk + 1), total), blk + 1 == nb);
        if (out) st_words_to_bytes(h, out);
    }
    __syncwarp();
}

// Absorb n <= 8 field elements; lane l < n contributes `mine` (Montgomery).  The canonical bytes are
// also written to copy_out (global, may be null).  All 32 lanes of the warp must call.
static __device__ __noinline__ void fs_absorb_frs(FsScratch& s, const char* tag, fr_t mine, int n, uint8_t* copy_out) {
    const int lane = threadIdx.x & 31;
    if (lane < n) {
        uint8_t tmp[32];
        fr_to_bytes(mine, tmp);
        for (int k = 0; k < 32; k++) s.pay[32 * lane + k] = tmp[k];
        if (copy_out)
            for (int k = 0; k < 32; k++) copy_out[32 * lane + k] = tmp[k];
    }
    __syncwarp();
    fs_hash_msg(s, 0, 0x01, tag, zk_strlen(tag), true, s.pay, 32u * n, 0, s.st);
}

// Absorb raw bytes (len <= 256) from any memory space; all lanes call.
__device__ inline void fs_absorb_bytes(FsScratch& s, const char* tag, const uint8_t* msg, uint32_t len) {
    const int lane = threadIdx.x & 31;
    for (uint32_t i = lane; i < len; i += 32) s.pay[i] = msg[i];
    __syncwarp();
    fs_hash_msg(s, 0, 0x01, tag, zk_strlen(tag), true, s.pay, len, 0, s.st);
}

// challenge state update (lane 0), the two squeeze hashes (lanes 0 / 1, in parallel), the four
// half-reductions (lanes 0-3).  Returns the Montgomery challenge on every lane (and s.rc = canonical).
static __device__ __noinline__ fr_t fs_challenge(FsScratch& s, const char* tag) {
    const int lane = threadIdx.x & 31;
    fs_hash_msg(s, 0, 0x02, tag, zk_strlen(tag), false, nullptr, 0, 0, s.st);
    // squeeze messages st || k (33 bytes, one block each) built by all lanes, hashed by lanes 0 and 1
    for (int k = 0; k < 2; k++) {
        uint8_t* b = reinterpret_cast<uint8_t*>(s.buf[k]);
        for (uint32_t p = lane; p < 64; p += 32) b[p] = p < 32 ? s.st[p] : p == 32 ? (uint8_t)k : 0;
    }
    __syncwarp();
    if (lane < 2) {
        uint32_t h[8];
        hash_init(h);
        hash_compress(h, s.buf[lane], 33, true);
        // the digest bytes as a little-endian 256-bit integer: limb i = word i
        fr_t x;
        for (int i = 0; i < 8; i++) x.v[i] = h[i];
        s.half[lane] = x;   // lane 0: lo, lane 1: hi
    }
    __syncwarp();
    if (lane < 4) {
        // lane 0: mont part of lo (R^2 lo), lane 1: mont part of hi 2^256 (R^3 hi), lane 2: canonical
        // hi 2^256 mod p (R^2 hi), lane 3: canonical lo mod p (lo < 2^256 < 3p).  One converged product
        // call for lanes 0-2 (three divergent calls serialised: ~3000 cycles per challenge)
        const fr_t lo = s.half[0], hi = s.half[1];
        const fr_t x = lane == 1 ? ZK_R3 : ZK_R2, y = lane == 0 ? lo : hi;
        const fr_t pv = fr_mul_cold(x, y);
        s.part[lane] = lane == 3 ? fr_reduce_once(fr_reduce_once(lo)) : pv;
    }
    __syncwarp();
    if (lane == 0) {
        s.r = fr_add(s.part[0], s.part[1]);
        s.rc = fr_add(s.part[2], s.part[3]);
    }
    __syncwarp();
    return s.r;
}

// Lagrange interpolation of the degree-d polynomial with values e[0..d] at 0..d, evaluated at x (d <= 3).
// The integer denominators are +-1, +-2, +-6; their inverses are constants (Montgomery form).
#define ZK_INV2 fr_const(0xffffffffu, 0x00000000u, 0x0001a401u, 0xac425bfdu, 0xf65e27fau, 0xccc627f7u, 0xd66282b7u, 0x0c1258acu)
#define ZK_INV6 fr_const(0xaaaaaaabu, 0xffffffffu, 0x5554c954u, 0x1be9e156u, 0xade09d57u, 0x11134802u, 0x63347f18u, 0x514f37c6u)
__device__ inline fr_t interp_small(const fr_t* e, int d, const fr_t& x) {
    fr_t xm[4];
    for (int j = 0; j <= d; j++) xm[j] = fr_sub(x, fr_from_u32((uint32_t)j));   // x - j
    fr_t acc = fr_zero();
    for (int i = 0; i <= d; i++) {
        fr_t num = fr_one();
        int den = 1;
        for (int j = 0; j <= d; j++) {
            if (j == i) continue;
            num = fr_mul_cold(num, xm[j]);
            den *= (i - j);
        }
        int ad = den < 0 ? -den : den;
        fr_t term = fr_mul_cold(e[i], num);
        if (ad == 2) term = fr_mul_cold(term, ZK_INV2);
        else if (ad == 6) term = fr_mul_cold(term, ZK_INV6);
        acc = den < 0 ? fr_sub(acc, term) : fr_add(acc, term);
    }
    return acc;
}

}  // namespace zk
