// transcript.cuh — device-resident Fiat-Shamir transcript (D3).
//
// The paper's protocols are interactive ("chosen by the verifier"); the
// challenges here come from a SHA-256 transcript whose 32-byte state lives in
// device memory so a whole sumcheck runs without a host round trip:
//   st0            = SHA256("zkdl-b200/v1/init" || seed32)
//   absorb(tag, m) : st = SHA256(st || 0x01 || u8(|tag|) || tag || u64be(|m|) || m)
//   challenge(tag) : st = SHA256(st || 0x02 || u8(|tag|) || tag)
//                    x  = LE512(SHA256(st || 0x00) || SHA256(st || 0x01)) mod p
//
// Latency matters (one transcript step per sumcheck round), so the step runs on one WARP of the
// finalizing block: messages are assembled in shared memory and hashed word-wise with the round
// function fully unrolled in registers; the field elements of a message are canonicalised by
// parallel lanes; the two squeeze hashes and the four half-reductions of the 512-bit challenge
// run on separate lanes.  x = lo + hi 2^256:  mont(x) = mont_mul(R^2, lo) + mont_mul(R^3, hi),
// canonical(x) = (lo mod p) + mont_mul(R^2, hi).
#pragma once
#include "fr.cuh"

namespace zk {

__device__ __constant__ static const uint32_t SHA_K[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }
__device__ __forceinline__ uint32_t ror32(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

struct Sha8 {
    uint32_t h[8];
};

// One compression of a 64-byte block given as 16 little-endian-loaded words (byte-swapped here).
// Fully unrolled so the round constants are immediates (a rolled loop with constant-bank loads ran
// at ~66 cycles/round on the B200); one out-of-line copy (~1K instructions) for the cold paths.
#define ZK_SHA_R(a, b, c, d, e, f, g, h, k, wv)                                                        \
    do {                                                                                               \
        const uint32_t t1_ = h + (ror32(e, 6) ^ ror32(e, 11) ^ ror32(e, 25)) + ((e & f) ^ (~e & g)) + (k) + (wv); \
        const uint32_t t2_ = (ror32(a, 2) ^ ror32(a, 13) ^ ror32(a, 22)) + ((a & b) ^ (a & c) ^ (b & c)); \
        d += t1_;                                                                                      \
        h = t1_ + t2_;                                                                                 \
    } while (0)
#define ZK_SHA_W(w, i)                                                                                 \
    (w[(i) & 15] += (ror32(w[((i) + 14) & 15], 17) ^ ror32(w[((i) + 14) & 15], 19) ^ (w[((i) + 14) & 15] >> 10)) + \
                    w[((i) + 9) & 15] +                                                                \
                    (ror32(w[((i) + 1) & 15], 7) ^ ror32(w[((i) + 1) & 15], 18) ^ (w[((i) + 1) & 15] >> 3)))
static __device__ __noinline__ Sha8 sha256_compress_s(Sha8 s, const uint32_t* blk) {
    static constexpr uint32_t K[64] = {
        0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
        0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
        0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
        0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
        0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
        0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
        0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
        0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; i++) w[i] = bswap32(blk[i]);
    uint32_t a = s.h[0], b = s.h[1], c = s.h[2], d = s.h[3], e = s.h[4], f = s.h[5], g = s.h[6], h = s.h[7];
#pragma unroll
    for (int i = 0; i < 64; i += 8) {
        if (i >= 16) {
#pragma unroll
            for (int q = 0; q < 8; q++) ZK_SHA_W(w, i + q);
        }
        ZK_SHA_R(a, b, c, d, e, f, g, h, K[i + 0], w[(i + 0) & 15]);
        ZK_SHA_R(h, a, b, c, d, e, f, g, K[i + 1], w[(i + 1) & 15]);
        ZK_SHA_R(g, h, a, b, c, d, e, f, K[i + 2], w[(i + 2) & 15]);
        ZK_SHA_R(f, g, h, a, b, c, d, e, K[i + 3], w[(i + 3) & 15]);
        ZK_SHA_R(e, f, g, h, a, b, c, d, K[i + 4], w[(i + 4) & 15]);
        ZK_SHA_R(d, e, f, g, h, a, b, c, K[i + 5], w[(i + 5) & 15]);
        ZK_SHA_R(c, d, e, f, g, h, a, b, K[i + 6], w[(i + 6) & 15]);
        ZK_SHA_R(b, c, d, e, f, g, h, a, K[i + 7], w[(i + 7) & 15]);
    }
    s.h[0] += a; s.h[1] += b; s.h[2] += c; s.h[3] += d; s.h[4] += e; s.h[5] += f; s.h[6] += g; s.h[7] += h;
    return s;
}
__device__ __forceinline__ void sha256_compress(uint32_t h[8], const uint32_t* blk) {
    Sha8 s;
#pragma unroll
    for (int i = 0; i < 8; i++) s.h[i] = h[i];
    s = sha256_compress_s(s, blk);
#pragma unroll
    for (int i = 0; i < 8; i++) h[i] = s.h[i];
}

// SHA-256 of n bytes held in a 4-byte-aligned buffer with room for the padding
// (capacity >= round_up(n + 9, 64)); the buffer is padded in place.  out: digest words (BE values).
__device__ inline void sha256_buf(uint8_t* buf, uint32_t n, uint32_t out[8]) {
    uint32_t total = (n + 9 + 63) & ~63u;
    buf[n] = 0x80;
    for (uint32_t i = n + 1; i < total - 8; i++) buf[i] = 0;
    const uint64_t bits = (uint64_t)n * 8;
    for (int i = 0; i < 8; i++) buf[total - 8 + i] = (uint8_t)(bits >> (56 - 8 * i));
    uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(buf);
    for (uint32_t blk = 0; blk < total / 64; blk++) sha256_compress(h, wp + 16 * blk);
#pragma unroll
    for (int i = 0; i < 8; i++) out[i] = h[i];
}

__device__ __forceinline__ uint32_t zk_strlen(const char* s) {
    uint32_t n = 0;
    while (s[n]) n++;
    return n;
}

// digest words <-> the 32 state bytes
__device__ __forceinline__ void st_words_to_bytes(const uint32_t w[8], uint8_t* out) {
    for (int i = 0; i < 8; i++) {
        out[4 * i] = (uint8_t)(w[i] >> 24);
        out[4 * i + 1] = (uint8_t)(w[i] >> 16);
        out[4 * i + 2] = (uint8_t)(w[i] >> 8);
        out[4 * i + 3] = (uint8_t)w[i];
    }
}

// Canonical 32-byte little-endian encoding of a Montgomery element.
__device__ inline void fr_to_bytes(const fr_t& a, uint8_t* out) {
    fr_t c = fr_to_canonical_cold(a);
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
// Shared scratch of one finalizing warp.
struct FsScratch {
    uint32_t buf[2][80];   // two 320-byte message buffers
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

// The 32 lanes assemble the padded message  st || dom || u8(|tag|) || tag || [u64be(plen)] || payload
// into s.buf[which] (each lane a strided subset of the bytes), then lane `hasher` compresses it and
// writes the digest to `out` (state bytes).  Every lane of the warp must call.
__device__ inline void fs_hash_msg(FsScratch& s, int which, uint8_t dom, const char* tag, uint32_t tl, bool with_len,
                                   const uint8_t* pay, uint32_t plen, int hasher, uint8_t* out) {
    const int lane = threadIdx.x & 31;
    uint8_t* b = reinterpret_cast<uint8_t*>(s.buf[which]);
    const uint32_t hl = 34 + tl + (with_len ? 8 : 0);
    const uint32_t total = hl + plen;
    const uint32_t padded = (total + 9 + 63) & ~63u;
    const uint64_t bits = (uint64_t)total * 8;
    for (uint32_t p = lane; p < padded; p += 32) {
        uint8_t v;
        if (p < 32) v = s.st[p];
        else if (p == 32) v = dom;
        else if (p == 33) v = (uint8_t)tl;
        else if (p < 34 + tl) v = (uint8_t)tag[p - 34];
        else if (p < hl) v = (uint8_t)((uint64_t)plen >> (56 - 8 * (p - 34 - tl)));
        else if (p < total) v = pay[p - hl];
        else if (p == total) v = 0x80;
        else if (p >= padded - 8) v = (uint8_t)(bits >> (56 - 8 * (p - (padded - 8))));
        else v = 0;
        b[p] = v;
    }
    __syncwarp();
    if (lane == hasher) {
        uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
        for (uint32_t blk = 0; blk < padded / 64; blk++) sha256_compress(h, s.buf[which] + 16 * blk);
        if (out) st_words_to_bytes(h, out);
    }
    __syncwarp();
}

// Absorb n <= 8 field elements; lane l < n contributes `mine` (Montgomery).  The canonical bytes are
// also written to copy_out (global, may be null).  All 32 lanes of the warp must call.
__device__ inline void fs_absorb_frs(FsScratch& s, const char* tag, const fr_t& mine, int n, uint8_t* copy_out) {
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
__device__ inline fr_t fs_challenge(FsScratch& s, const char* tag) {
    const int lane = threadIdx.x & 31;
    fs_hash_msg(s, 0, 0x02, tag, zk_strlen(tag), false, nullptr, 0, 0, s.st);
    // squeeze messages st || k (33 bytes, one block each) built by all lanes, hashed by lanes 0 and 1
    for (int k = 0; k < 2; k++) {
        uint8_t* b = reinterpret_cast<uint8_t*>(s.buf[k]);
        for (uint32_t p = lane; p < 64; p += 32) {
            uint8_t v;
            if (p < 32) v = s.st[p];
            else if (p == 32) v = (uint8_t)k;
            else if (p == 33) v = 0x80;
            else if (p == 62) v = (uint8_t)((33 * 8) >> 8);
            else if (p == 63) v = (uint8_t)(33 * 8);
            else v = 0;
            b[p] = v;
        }
    }
    __syncwarp();
    if (lane < 2) {
        uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
        sha256_compress(h, s.buf[lane]);
        // digest bytes are h[i] big-endian; as a little-endian 256-bit integer limb i = bytes 4i..4i+3
        fr_t x;
        for (int i = 0; i < 8; i++) x.v[i] = bswap32(h[i]);
        s.half[lane] = x;   // lane 0: lo, lane 1: hi
    }
    __syncwarp();
    if (lane < 4) {
        const fr_t lo = s.half[0], hi = s.half[1];
        fr_t v;
        if (lane == 0) v = fr_mul_cold(ZK_R2, lo);          // mont part of lo
        else if (lane == 1) v = fr_mul_cold(ZK_R3, hi);     // mont part of hi * 2^256
        else if (lane == 2) v = fr_mul_cold(ZK_R2, hi);     // canonical hi * 2^256 mod p
        else v = fr_reduce_once(fr_reduce_once(lo));   // canonical lo mod p (lo < 2^256 < 3p)
        s.part[lane] = v;
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
