// transcript.cuh — device-resident Fiat-Shamir transcript (D3).
//
// The paper's protocols are interactive ("chosen by the verifier"); the
// challenges here come from a SHA-256 transcript whose 32-byte state lives in
// device memory so a whole sumcheck runs without a host round trip:
//   st0            = SHA256("zkdl-b200/v1/init" || seed32)
//   absorb(tag, m) : st = SHA256(st || 0x01 || u8(|tag|) || tag || u64be(|m|) || m)
//   challenge(tag) : st = SHA256(st || 0x02 || u8(|tag|) || tag)
//                    x  = LE512(SHA256(st || 0x00) || SHA256(st || 0x01)) mod p
// All functions here run on ONE thread (the finalizing thread of a kernel).
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

struct Sha256 {
    uint32_t h[8];
    uint8_t buf[64];
    uint32_t nbuf;
    uint64_t len;

    __device__ __forceinline__ static uint32_t ror(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

    __device__ void init() {
        h[0] = 0x6a09e667; h[1] = 0xbb67ae85; h[2] = 0x3c6ef372; h[3] = 0xa54ff53a;
        h[4] = 0x510e527f; h[5] = 0x9b05688c; h[6] = 0x1f83d9ab; h[7] = 0x5be0cd19;
        nbuf = 0;
        len = 0;
    }
    __device__ void block(const uint8_t* p) {
        uint32_t w[16];
#pragma unroll
        for (int i = 0; i < 16; i++)
            w[i] = ((uint32_t)p[4 * i] << 24) | ((uint32_t)p[4 * i + 1] << 16) | ((uint32_t)p[4 * i + 2] << 8) | p[4 * i + 3];
        uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
#pragma unroll
        for (int i = 0; i < 64; i++) {
            uint32_t wi;
            if (i < 16) {
                wi = w[i];
            } else {
                uint32_t w15 = w[(i - 15) & 15], w2 = w[(i - 2) & 15];
                uint32_t s0 = ror(w15, 7) ^ ror(w15, 18) ^ (w15 >> 3);
                uint32_t s1 = ror(w2, 17) ^ ror(w2, 19) ^ (w2 >> 10);
                wi = w[i & 15] + s0 + w[(i - 7) & 15] + s1;
                w[i & 15] = wi;
            }
            uint32_t S1 = ror(e, 6) ^ ror(e, 11) ^ ror(e, 25);
            uint32_t ch = (e & f) ^ (~e & g);
            uint32_t t1 = hh + S1 + ch + SHA_K[i] + wi;
            uint32_t S0 = ror(a, 2) ^ ror(a, 13) ^ ror(a, 22);
            uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
            uint32_t t2 = S0 + mj;
            hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
        }
        h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
    }
    __device__ void update(const uint8_t* p, uint64_t n) {
        len += n;
        while (n) {
            uint32_t take = 64 - nbuf;
            if (take > n) take = (uint32_t)n;
            for (uint32_t i = 0; i < take; i++) buf[nbuf + i] = p[i];
            nbuf += take;
            p += take;
            n -= take;
            if (nbuf == 64) {
                block(buf);
                nbuf = 0;
            }
        }
    }
    __device__ void update_byte(uint8_t b) { update(&b, 1); }
    __device__ void final(uint8_t out[32]) {
        uint64_t bits = len * 8;
        update_byte(0x80);
        while (nbuf != 56) update_byte(0);
        uint8_t lb[8];
        for (int i = 0; i < 8; i++) lb[i] = (uint8_t)(bits >> (56 - 8 * i));
        update(lb, 8);
        for (int i = 0; i < 8; i++) {
            out[4 * i] = (uint8_t)(h[i] >> 24);
            out[4 * i + 1] = (uint8_t)(h[i] >> 16);
            out[4 * i + 2] = (uint8_t)(h[i] >> 8);
            out[4 * i + 3] = (uint8_t)h[i];
        }
    }
};

__device__ __forceinline__ uint32_t zk_strlen(const char* s) {
    uint32_t n = 0;
    while (s[n]) n++;
    return n;
}

// Canonical 32-byte little-endian encoding of a Montgomery element.
__device__ inline void fr_to_bytes(const fr_t& a, uint8_t out[32]) {
    fr_t c = fr_to_canonical(a);
    for (int i = 0; i < 8; i++) {
        out[4 * i] = (uint8_t)c.v[i];
        out[4 * i + 1] = (uint8_t)(c.v[i] >> 8);
        out[4 * i + 2] = (uint8_t)(c.v[i] >> 16);
        out[4 * i + 3] = (uint8_t)(c.v[i] >> 24);
    }
}

__device__ inline void tr_init(uint8_t* st, const uint8_t seed[32]) {
    Sha256 s;
    s.init();
    const char* lbl = "zkdl-b200/v1/init";
    s.update((const uint8_t*)lbl, zk_strlen(lbl));
    s.update(seed, 32);
    s.final(st);
}

__device__ inline void tr_absorb_begin(Sha256& s, const uint8_t* st, const char* tag, uint64_t len) {
    s.init();
    s.update(st, 32);
    s.update_byte(0x01);
    uint32_t tl = zk_strlen(tag);
    s.update_byte((uint8_t)tl);
    s.update((const uint8_t*)tag, tl);
    uint8_t lb[8];
    for (int i = 0; i < 8; i++) lb[i] = (uint8_t)(len >> (56 - 8 * i));
    s.update(lb, 8);
}

__device__ inline void tr_absorb(uint8_t* st, const char* tag, const uint8_t* msg, uint64_t len) {
    Sha256 s;
    tr_absorb_begin(s, st, tag, len);
    s.update(msg, len);
    s.final(st);
}

// absorb n field elements (Montgomery in registers/memory) as canonical LE bytes
__device__ inline void tr_absorb_frs(uint8_t* st, const char* tag, const fr_t* v, int n, uint8_t* copy_out = nullptr) {
    Sha256 s;
    tr_absorb_begin(s, st, tag, 32ull * n);
    for (int i = 0; i < n; i++) {
        uint8_t b[32];
        fr_to_bytes(v[i], b);
        s.update(b, 32);
        if (copy_out)
            for (int k = 0; k < 32; k++) copy_out[32 * i + k] = b[k];
    }
    s.final(st);
}

// challenge: returns the Montgomery form of the squeezed element
__device__ inline fr_t tr_challenge(uint8_t* st, const char* tag) {
    Sha256 s;
    s.init();
    s.update(st, 32);
    s.update_byte(0x02);
    uint32_t tl = zk_strlen(tag);
    s.update_byte((uint8_t)tl);
    s.update((const uint8_t*)tag, tl);
    s.final(st);
    uint8_t h[64];
    for (int k = 0; k < 2; k++) {
        s.init();
        s.update(st, 32);
        s.update_byte((uint8_t)k);
        s.final(h + 32 * k);
    }
    // x = lo + hi * 2^256 with lo, hi < 2^256;  mont(x) = lo*R + hi*R^2 = mont_mul(R2, lo) + mont_mul(R3, hi)
    fr_t lo, hi;
    for (int i = 0; i < 8; i++) {
        lo.v[i] = (uint32_t)h[4 * i] | ((uint32_t)h[4 * i + 1] << 8) | ((uint32_t)h[4 * i + 2] << 16) |
                  ((uint32_t)h[4 * i + 3] << 24);
        hi.v[i] = (uint32_t)h[32 + 4 * i] | ((uint32_t)h[32 + 4 * i + 1] << 8) | ((uint32_t)h[32 + 4 * i + 2] << 16) |
                  ((uint32_t)h[32 + 4 * i + 3] << 24);
    }
    return fr_add(fr_mul(ZK_R2, lo), fr_mul(ZK_R3, hi));
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
            num = fr_mul(num, xm[j]);
            den *= (i - j);
        }
        int ad = den < 0 ? -den : den;
        fr_t term = fr_mul(e[i], num);
        if (ad == 2) term = fr_mul(term, ZK_INV2);
        else if (ad == 6) term = fr_mul(term, ZK_INV6);
        acc = den < 0 ? fr_sub(acc, term) : fr_add(acc, term);
    }
    return acc;
}

}  // namespace zk
