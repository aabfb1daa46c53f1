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
// Out of line and rolled 4 x 16 rounds: the transcript runs on cold code paths (see fr_mul_cold).
static __device__ __noinline__ Sha8 sha256_compress_s(Sha8 s, const uint32_t* blk) {
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; i++) w[i] = bswap32(blk[i]);
    uint32_t a = s.h[0], b = s.h[1], c = s.h[2], d = s.h[3], e = s.h[4], f = s.h[5], g = s.h[6], hh = s.h[7];
#pragma unroll 1
    for (int j = 0; j < 64; j += 16) {
#pragma unroll
        for (int i = 0; i < 16; i++) {
            uint32_t wi;
            if (j == 0) {
                wi = w[i];
            } else {
                const uint32_t w15 = w[(i + 1) & 15], w2 = w[(i + 14) & 15];
                const uint32_t s0 = ror32(w15, 7) ^ ror32(w15, 18) ^ (w15 >> 3);
                const uint32_t s1 = ror32(w2, 17) ^ ror32(w2, 19) ^ (w2 >> 10);
                wi = w[i] + s0 + w[(i + 9) & 15] + s1;
                w[i] = wi;
            }
            const uint32_t S1 = ror32(e, 6) ^ ror32(e, 11) ^ ror32(e, 25);
            const uint32_t ch = (e & f) ^ (~e & g);
            const uint32_t t1 = hh + S1 + ch + SHA_K[j + i] + wi;
            const uint32_t S0 = ror32(a, 2) ^ ror32(a, 13) ^ ror32(a, 22);
            const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
            hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + S0 + mj;
        }
    }
    s.h[0] += a; s.h[1] += b; s.h[2] += c; s.h[3] += d; s.h[4] += e; s.h[5] += f; s.h[6] += g; s.h[7] += hh;
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
    fr_t part[4];
    fr_t r;
    fr_t rc;               // canonical r
};

// lane 0 copies the global state in / out
__device__ __forceinline__ void fs_begin(FsScratch& s, const uint8_t* st_g) {
    if ((threadIdx.x & 31) == 0)
        for (int i = 0; i < 32; i++) s.st[i] = st_g[i];
    __syncwarp();
}
__device__ __forceinline__ void fs_end(FsScratch& s, uint8_t* st_g) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0)
        for (int i = 0; i < 32; i++) st_g[i] = s.st[i];
    __syncwarp();
}

// header of an absorb: st || 0x01 || u8(|tag|) || tag || u64be(len); returns its length
__device__ inline uint32_t fs_absorb_header(FsScratch& s, uint8_t* b, const char* tag, uint64_t len) {
    for (int i = 0; i < 32; i++) b[i] = s.st[i];
    uint32_t tl = zk_strlen(tag);
    b[32] = 0x01;
    b[33] = (uint8_t)tl;
    for (uint32_t i = 0; i < tl; i++) b[34 + i] = (uint8_t)tag[i];
    for (int i = 0; i < 8; i++) b[34 + tl + i] = (uint8_t)(len >> (56 - 8 * i));
    return 42 + tl;
}

// Absorb n <= 8 field elements; lane l < n contributes `mine` (Montgomery).  The canonical bytes are
// also written to copy_out (global, may be null).  All 32 lanes of the warp must call.
__device__ inline void fs_absorb_frs(FsScratch& s, const char* tag, const fr_t& mine, int n, uint8_t* copy_out) {
    const int lane = threadIdx.x & 31;
    uint8_t* b = reinterpret_cast<uint8_t*>(s.buf[0]);
    __shared__ uint32_t hlen_sm;
    if (lane == 0) hlen_sm = fs_absorb_header(s, b, tag, 32ull * n);
    __syncwarp();
    const uint32_t hl = hlen_sm;
    if (lane < n) {
        uint8_t tmp[32];
        fr_to_bytes(mine, tmp);
        for (int k = 0; k < 32; k++) b[hl + 32 * lane + k] = tmp[k];
        if (copy_out)
            for (int k = 0; k < 32; k++) copy_out[32 * lane + k] = tmp[k];
    }
    __syncwarp();
    if (lane == 0) {
        uint32_t d[8];
        sha256_buf(b, hl + 32 * n, d);
        st_words_to_bytes(d, s.st);
    }
    __syncwarp();
}

// Absorb raw bytes (lane 0 only does the work; all lanes call).  len <= 256.
__device__ inline void fs_absorb_bytes(FsScratch& s, const char* tag, const uint8_t* msg, uint32_t len) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
        uint8_t* b = reinterpret_cast<uint8_t*>(s.buf[0]);
        uint32_t hl = fs_absorb_header(s, b, tag, len);
        for (uint32_t i = 0; i < len; i++) b[hl + i] = msg[i];
        uint32_t d[8];
        sha256_buf(b, hl + len, d);
        st_words_to_bytes(d, s.st);
    }
    __syncwarp();
}

// lane 0: the challenge state update; lanes 0/1: the two squeeze hashes; lanes 0-3: the four
// half-reductions.  Returns the Montgomery challenge on every lane (and s.rc = canonical).
__device__ inline fr_t fs_challenge(FsScratch& s, const char* tag) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
        uint8_t* b = reinterpret_cast<uint8_t*>(s.buf[0]);
        for (int i = 0; i < 32; i++) b[i] = s.st[i];
        uint32_t tl = zk_strlen(tag);
        b[32] = 0x02;
        b[33] = (uint8_t)tl;
        for (uint32_t i = 0; i < tl; i++) b[34 + i] = (uint8_t)tag[i];
        uint32_t d[8];
        sha256_buf(b, 34 + tl, d);
        st_words_to_bytes(d, s.st);
    }
    __syncwarp();
    __shared__ fr_t half[2];
    if (lane < 2) {
        uint8_t* b = reinterpret_cast<uint8_t*>(s.buf[lane]);
        for (int i = 0; i < 32; i++) b[i] = s.st[i];
        b[32] = (uint8_t)lane;
        uint32_t d[8];
        sha256_buf(b, 33, d);
        // digest bytes are d[i] big-endian; as a little-endian 256-bit integer limb i = bytes 4i..4i+3
        fr_t x;
        for (int i = 0; i < 8; i++) x.v[i] = bswap32(d[i]);
        half[lane] = x;   // lane 0: lo, lane 1: hi
    }
    __syncwarp();
    if (lane < 4) {
        const fr_t lo = half[0], hi = half[1];
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
