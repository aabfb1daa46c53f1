// verify.cu — host verifiers for the proofs libzkdl emits (D23).
//
// "The verification time is almost the same as the proving time because the verifier has to
// process the same sequence of sumcheck rounds": verification is a sequential replay
// of the Fiat-Shamir transcript (D3) with O(deg) field operations per round, so it runs on the
// host.  Everything here is plain host C++ with its own field arithmetic (4 x 64-bit Montgomery,
// R = 2^256) and its own BLAKE2s (RFC 7693); no device, no context.  The verifiers check every
// round identity and the final identity of each protocol; the finals themselves are claims on the
// committed tensors (commitments are out of scope) and are returned to the caller.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "zkdl.h"

namespace {

typedef unsigned __int128 u128;

// ------------------------------------------------------------------ Fr, 4 x 64-bit Montgomery
struct F {
    uint64_t v[4];
};
const uint64_t P[4] = {0xFFFFFFFF00000001ull, 0x53BDA402FFFE5BFEull, 0x3339D80809A1D805ull, 0x73EDA753299D7D48ull};

bool geq_p(const uint64_t a[4]) {
    for (int i = 3; i >= 0; i--) {
        if (a[i] != P[i]) return a[i] > P[i];
    }
    return true;
}
void sub_p(uint64_t a[4]) {
    uint64_t br = 0;
    for (int i = 0; i < 4; i++) {
        const u128 d = (u128)a[i] - P[i] - br;
        a[i] = (uint64_t)d;
        br = (uint64_t)(d >> 64) ? 1 : 0;
    }
}
F add(const F& a, const F& b) {
    F r;
    uint64_t c = 0;
    for (int i = 0; i < 4; i++) {
        const u128 s = (u128)a.v[i] + b.v[i] + c;
        r.v[i] = (uint64_t)s;
        c = (uint64_t)(s >> 64);
    }
    if (c || geq_p(r.v)) sub_p(r.v);
    return r;
}
F sub(const F& a, const F& b) {
    F r;
    uint64_t br = 0;
    for (int i = 0; i < 4; i++) {
        const u128 d = (u128)a.v[i] - b.v[i] - br;
        r.v[i] = (uint64_t)d;
        br = (uint64_t)(d >> 64) ? 1 : 0;
    }
    if (br) {   // add p back
        uint64_t c = 0;
        for (int i = 0; i < 4; i++) {
            const u128 s = (u128)r.v[i] + P[i] + c;
            r.v[i] = (uint64_t)s;
            c = (uint64_t)(s >> 64);
        }
    }
    return r;
}
uint64_t NP;   // -p^{-1} mod 2^64
F R2;          // 2^512 mod p (Montgomery form of 2^256)
F ONE;         // Montgomery form of 1 (= 2^256 mod p)
// CIOS Montgomery product a b 2^-256 mod p
F mul(const F& a, const F& b) {
    uint64_t t[6] = {0, 0, 0, 0, 0, 0};
    for (int i = 0; i < 4; i++) {
        uint64_t c = 0;
        for (int j = 0; j < 4; j++) {
            const u128 s = (u128)a.v[j] * b.v[i] + t[j] + c;
            t[j] = (uint64_t)s;
            c = (uint64_t)(s >> 64);
        }
        u128 s = (u128)t[4] + c;
        t[4] = (uint64_t)s;
        t[5] = (uint64_t)(s >> 64);
        const uint64_t m = t[0] * NP;
        s = (u128)m * P[0] + t[0];
        c = (uint64_t)(s >> 64);
        for (int j = 1; j < 4; j++) {
            s = (u128)m * P[j] + t[j] + c;
            t[j - 1] = (uint64_t)s;
            c = (uint64_t)(s >> 64);
        }
        s = (u128)t[4] + c;
        t[3] = (uint64_t)s;
        t[4] = t[5] + (uint64_t)(s >> 64);
    }
    F r = {{t[0], t[1], t[2], t[3]}};
    if (t[4] || geq_p(r.v)) sub_p(r.v);
    return r;
}
bool init_done = false;
void init() {
    if (init_done) return;
    uint64_t x = 1;   // Newton: x = p0^{-1} mod 2^64
    for (int i = 0; i < 7; i++) x *= 2 - P[0] * x;
    NP = 0 - x;
    F r = {{1, 0, 0, 0}};   // 2^512 mod p by 512 doublings of 1 (plain integers)
    for (int i = 0; i < 512; i++) {
        r = add(r, r);
        if (i == 255) ONE = r;
    }
    R2 = r;
    init_done = true;
}
F zero() { return F{{0, 0, 0, 0}}; }
bool eq(const F& a, const F& b) { return !memcmp(a.v, b.v, 32); }
F from_u64(uint64_t x) { return mul(F{{x, 0, 0, 0}}, R2); }
F neg(const F& a) { return sub(zero(), a); }
// canonical little-endian bytes <-> Montgomery form; false if >= p
bool load(const uint8_t* b, F& out) {
    uint64_t w[4];
    memcpy(w, b, 32);
    if (geq_p(w)) return false;
    F x;
    memcpy(x.v, w, 32);
    out = mul(x, R2);
    return true;
}
void store(const F& a, uint8_t* b) {
    const F x = mul(a, F{{1, 0, 0, 0}});
    memcpy(b, x.v, 32);
}
F pow(F a, const uint64_t e[4]) {
    F r = ONE;
    for (int i = 3; i >= 0; i--)
        for (int k = 63; k >= 0; k--) {
            r = mul(r, r);
            if ((e[i] >> k) & 1) r = mul(r, a);
        }
    return r;
}
F inv(const F& a) {
    uint64_t e[4] = {P[0] - 2, P[1], P[2], P[3]};
    return pow(a, e);
}
F one_minus(const F& a) { return sub(ONE, a); }
// beta(u, v) = prod_t (u_t v_t + (1 - u_t)(1 - v_t))
F beta(const F* u, const F* v, uint32_t k) {
    F acc = ONE;
    for (uint32_t t = 0; t < k; t++) acc = mul(acc, add(mul(u[t], v[t]), mul(one_minus(u[t]), one_minus(v[t]))));
    return acc;
}
// beta(u, bits of b), LSB-first (D2)
F beta_at(const F* u, uint32_t k, uint64_t b) {
    F acc = ONE;
    for (uint32_t t = 0; t < k; t++) acc = mul(acc, ((b >> t) & 1) ? u[t] : one_minus(u[t]));
    return acc;
}
// the degree-d polynomial through (X, e[X]), X = 0..d, at x (Lagrange)
F interp(const F* e, int d, const F& x) {
    F acc = zero();
    for (int i = 0; i <= d; i++) {
        F num = ONE, den = ONE;
        for (int j = 0; j <= d; j++) {
            if (j == i) continue;
            num = mul(num, sub(x, from_u64((uint64_t)j)));
            den = mul(den, i > j ? from_u64((uint64_t)(i - j)) : neg(from_u64((uint64_t)(j - i))));
        }
        acc = add(acc, mul(e[i], mul(num, inv(den))));
    }
    return acc;
}

// ------------------------------------------------------------------ BLAKE2s-256 (RFC 7693)
struct B2s {
    uint32_t h[8];
    uint8_t buf[64];
    uint32_t t = 0, n = 0;   // bytes compressed, bytes buffered
};
const uint32_t IV[8] = {0x6A09E667u, 0xBB67AE85u, 0x3C6EF372u, 0xA54FF53Au,
                        0x510E527Fu, 0x9B05688Cu, 0x1F83D9ABu, 0x5BE0CD19u};
const uint8_t SIGMA[10][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0}};
inline uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }
void b2_compress(B2s& s, const uint8_t* blk, bool last) {
    uint32_t m[16], v[16];
    for (int i = 0; i < 16; i++)
        m[i] = (uint32_t)blk[4 * i] | (uint32_t)blk[4 * i + 1] << 8 | (uint32_t)blk[4 * i + 2] << 16 |
               (uint32_t)blk[4 * i + 3] << 24;
    for (int i = 0; i < 8; i++) {
        v[i] = s.h[i];
        v[i + 8] = IV[i];
    }
    v[12] ^= s.t;   // byte counter (messages < 2^32 bytes)
    if (last) v[14] = ~v[14];
    auto G = [&](int a, int b, int c, int d, uint32_t x, uint32_t y) {
        v[a] += v[b] + x; v[d] = rotr(v[d] ^ v[a], 16);
        v[c] += v[d];     v[b] = rotr(v[b] ^ v[c], 12);
        v[a] += v[b] + y; v[d] = rotr(v[d] ^ v[a], 8);
        v[c] += v[d];     v[b] = rotr(v[b] ^ v[c], 7);
    };
    for (int r = 0; r < 10; r++) {
        const uint8_t* g = SIGMA[r];
        G(0, 4, 8, 12, m[g[0]], m[g[1]]);
        G(1, 5, 9, 13, m[g[2]], m[g[3]]);
        G(2, 6, 10, 14, m[g[4]], m[g[5]]);
        G(3, 7, 11, 15, m[g[6]], m[g[7]]);
        G(0, 5, 10, 15, m[g[8]], m[g[9]]);
        G(1, 6, 11, 12, m[g[10]], m[g[11]]);
        G(2, 7, 8, 13, m[g[12]], m[g[13]]);
        G(3, 4, 9, 14, m[g[14]], m[g[15]]);
    }
    for (int i = 0; i < 8; i++) s.h[i] ^= v[i] ^ v[i + 8];
}
void b2_init(B2s& s) {
    for (int i = 0; i < 8; i++) s.h[i] = IV[i];
    s.h[0] ^= 0x01010020u;   // digest 32 bytes, no key, fanout 1, depth 1
    s.t = s.n = 0;
}
void b2_update(B2s& s, const void* data, uint64_t len) {
    const uint8_t* p = static_cast<const uint8_t*>(data);
    while (len) {
        if (s.n == 64) {   // a full buffer is compressed only once more input follows (the last block is special)
            s.t += 64;
            b2_compress(s, s.buf, false);
            s.n = 0;
        }
        const uint32_t k = (uint32_t)(len < 64 - s.n ? len : 64 - s.n);
        memcpy(s.buf + s.n, p, k);
        s.n += k;
        p += k;
        len -= k;
    }
}
void b2_final(B2s& s, uint8_t out[32]) {
    s.t += s.n;
    memset(s.buf + s.n, 0, 64 - s.n);
    b2_compress(s, s.buf, true);
    for (int i = 0; i < 8; i++)
        for (int k = 0; k < 4; k++) out[4 * i + k] = (uint8_t)(s.h[i] >> (8 * k));
}

// ------------------------------------------------------------------ transcript (D3)
void tr_absorb(uint8_t st[32], const char* tag, const void* msg, uint64_t len) {
    B2s s;
    b2_init(s);
    const uint8_t dom = 0x01, tl = (uint8_t)strlen(tag);
    uint8_t lb[8];
    for (int i = 0; i < 8; i++) lb[i] = (uint8_t)(len >> (56 - 8 * i));
    b2_update(s, st, 32);
    b2_update(s, &dom, 1);
    b2_update(s, &tl, 1);
    b2_update(s, tag, tl);
    b2_update(s, lb, 8);
    b2_update(s, msg, len);
    b2_final(s, st);
}
F tr_challenge(uint8_t st[32], const char* tag) {
    B2s s;
    b2_init(s);
    const uint8_t dom = 0x02, tl = (uint8_t)strlen(tag);
    b2_update(s, st, 32);
    b2_update(s, &dom, 1);
    b2_update(s, &tl, 1);
    b2_update(s, tag, tl);
    b2_final(s, st);
    uint8_t h[64];
    for (uint8_t k = 0; k < 2; k++) {
        b2_init(s);
        b2_update(s, st, 32);
        b2_update(s, &k, 1);
        b2_final(s, h + 32 * k);
    }
    // x = lo + hi 2^256 mod p: each half reduced below p (2^256 < 3p), then lo R + hi 2^256 R in Montgomery form
    F lo, hi;
    memcpy(lo.v, h, 32);
    memcpy(hi.v, h + 32, 32);
    while (geq_p(lo.v)) sub_p(lo.v);
    while (geq_p(hi.v)) sub_p(hi.v);
    return add(mul(lo, R2), mul(mul(hi, R2), R2));
}
void tr_absorb_frs(uint8_t st[32], const char* tag, const F* v, uint32_t n) {
    std::string b(32ull * n, '\0');
    for (uint32_t i = 0; i < n; i++) store(v[i], reinterpret_cast<uint8_t*>(&b[32ull * i]));
    tr_absorb(st, tag, b.data(), b.size());
}
void tr_absorb_u32s(uint8_t st[32], const char* tag, const uint32_t* w, uint32_t n) {
    uint8_t b[64];
    for (uint32_t i = 0; i < n; i++)
        for (int k = 0; k < 4; k++) b[4 * i + k] = (uint8_t)(w[i] >> (8 * k));
    tr_absorb(st, tag, b, 4ull * n);
}
uint32_t rd32(const uint8_t* p) { return (uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24; }

struct Reject {
    int32_t where;
};
struct Bad {
    zk_status st;
};
void need(bool ok, zk_status st = ZK_ERR_ARG) {
    if (!ok) throw Bad{st};
}
F ld(const uint8_t* b) {
    F x;
    need(load(b, x), ZK_ERR_NONCANONICAL);
    return x;
}

// The product sumcheck (Protocol 3 with the D4 message convention, D3c transcript): returns the
// point r; throws Reject{t + 1} for a failed round identity, Reject{-100} for the final identity.
void sumcheck_rounds(uint8_t st[32], uint32_t m, uint32_t n_eq, uint32_t K, const F* w, F c, const uint8_t* msgs,
                     const uint8_t* finals, F* r) {
    for (uint32_t t = 0; t < m; t++) {
        F ev[4];
        for (uint32_t X = 0; X <= K; X++) ev[X] = ld(msgs + 32ull * (t * (K + 1) + X));
        // f_t under the beta(w, .) factor (the prefix and beta(w_t, X) divided out), else g_t
        const F lhs = t < n_eq ? add(mul(one_minus(w[t]), ev[0]), mul(w[t], ev[1])) : add(ev[0], ev[1]);
        if (!eq(lhs, c)) throw Reject{(int32_t)t + 1};
        tr_absorb_frs(st, "sc/msg", ev, K + 1);
        r[t] = tr_challenge(st, "sc/r");
        c = interp(ev, (int)K, r[t]);
    }
    F fin[3], prod = ONE;
    for (uint32_t k = 0; k < K; k++) {
        fin[k] = ld(finals + 32ull * k);
        prod = mul(prod, fin[k]);
    }
    if (!eq(prod, c)) throw Reject{-100};
    tr_absorb_frs(st, "sc/final", fin, K);
}

template <class Fn>
zk_status guarded(int32_t* fail, Fn&& fn) {
    if (fail) *fail = 0;
    try {
        init();
        fn();
        return ZK_OK;
    } catch (const Reject& r) {
        if (fail) *fail = r.where;
        return ZK_REJECT;
    } catch (const Bad& b) {
        return b.st;
    } catch (...) {
        return ZK_ERR_INTERNAL;
    }
}
void out_points(const F* v, uint32_t n, zk_fr* out) {
    if (out)
        for (uint32_t i = 0; i < n; i++) store(v[i], out[i].b);
}

}  // namespace

extern "C" {

zk_status zk_htr_init(const uint8_t seed[32], uint8_t st[32]) {
    if (!seed || !st) return ZK_ERR_ARG;
    B2s s;
    b2_init(s);
    const char* lbl = "zkdl-b200/v1/init";
    b2_update(s, lbl, strlen(lbl));
    b2_update(s, seed, 32);
    b2_final(s, st);
    return ZK_OK;
}

zk_status zk_htr_absorb(uint8_t st[32], const char* tag, const void* msg, uint64_t len) {
    if (!st || !tag || strlen(tag) > 255 || (len && !msg)) return ZK_ERR_ARG;
    tr_absorb(st, tag, msg, len);
    return ZK_OK;
}

zk_status zk_htr_challenges(uint8_t st[32], const char* tag, uint32_t n, zk_fr* out) {
    if (!st || !tag || strlen(tag) > 255 || (n && !out)) return ZK_ERR_ARG;
    init();
    for (uint32_t i = 0; i < n; i++) store(tr_challenge(st, tag), out[i].b);
    return ZK_OK;
}

zk_status zk_verify_sumcheck(uint8_t st[32], const uint8_t* proof, uint64_t proof_len, const uint32_t expect[3],
                             const zk_fr* w, const zk_fr* claim, zk_fr* point_out, int32_t* fail) {
    return guarded(fail, [&] {
        need(st && proof && expect && proof_len >= 12);
        const uint32_t m = rd32(proof), n_eq = rd32(proof + 4), K = rd32(proof + 8);
        // the statement's shape is the verifier's, not the prover's: the header must match it
        if (m != expect[0] || n_eq != expect[1] || K != expect[2]) throw Reject{-2};
        need(m >= 1 && m <= 64 && n_eq <= m && K >= 1 && K <= 3 && (n_eq == 0 || w));
        need(proof_len == 12 + 32 + 32ull * m * (K + 1) + 32ull * K);
        F wf[64], r[64];
        for (uint32_t t = 0; t < n_eq; t++) wf[t] = ld(w[t].b);
        const F c = ld(proof + 12);
        if (claim && !eq(ld(claim->b), c)) throw Reject{-1};   // the proof is for another claim
        const uint32_t hdr[3] = {m, n_eq, K};
        tr_absorb_u32s(st, "sc/hdr", hdr, 3);
        tr_absorb_frs(st, "sc/claim", &c, 1);
        sumcheck_rounds(st, m, n_eq, K, wf, c, proof + 44, proof + 44 + 32ull * m * (K + 1), r);
        out_points(r, m, point_out);
    });
}

zk_status zk_verify_hadamard_zero(uint8_t st[32], const uint8_t* proof, uint64_t proof_len, uint32_t expect_m,
                                  zk_fr* w_out, zk_fr* point_out, int32_t* fail) {
    return guarded(fail, [&] {
        need(st && proof && proof_len >= 4);
        const uint32_t m = rd32(proof);
        if (m != expect_m) throw Reject{-2};
        need(m >= 1 && m <= 64 && proof_len == 4 + 96ull * m + 96);
        tr_absorb_u32s(st, "hd/hdr", &m, 1);
        F w[64], r[64];
        for (uint32_t t = 0; t < m; t++) w[t] = tr_challenge(st, "hd/w");
        F c = zero();   // Protocol 2: the zero statement sum_x beta(w, x) (Y - A B)(x) = 0
        const uint8_t* msgs = proof + 4;
        for (uint32_t t = 0; t < m; t++) {
            F ev[3];
            for (int X = 0; X < 3; X++) ev[X] = ld(msgs + 32ull * (3 * t + X));
            if (!eq(add(mul(one_minus(w[t]), ev[0]), mul(w[t], ev[1])), c)) throw Reject{(int32_t)t + 1};
            tr_absorb_frs(st, "sc/msg", ev, 3);
            r[t] = tr_challenge(st, "sc/r");
            c = interp(ev, 2, r[t]);
        }
        F fin[3];
        for (int k = 0; k < 3; k++) fin[k] = ld(msgs + 96ull * m + 32 * k);
        if (!eq(c, sub(fin[0], mul(fin[1], fin[2])))) throw Reject{-100};   // Y~(r) - A~(r) B~(r)
        tr_absorb_frs(st, "sc/final", fin, 3);
        out_points(w, m, w_out);
        out_points(r, m, point_out);
    });
}

// zkReLU (App. A; transcript D3b).  The final identity is the six statements of
// Eq. (zkrelu-*-sc) at the final point, with the verifier's own beta, s and s' evaluations.
zk_status zk_verify_relu(uint8_t st[32], const uint8_t* proof, uint64_t proof_len, const uint32_t expect[3],
                         const zk_fr* pts, zk_fr* point_out, int32_t* fail) {
    return guarded(fail, [&] {
        need(st && proof && expect && proof_len >= 12);
        const uint32_t logD = rd32(proof), Q = rd32(proof + 4), R = rd32(proof + 8);
        if (logD != expect[0] || Q != expect[1] || R != expect[2]) throw Reject{-2};
        need(logD >= 1 && logD <= 40 && Q >= 1 && R >= 1 && Q <= 32 && R <= 32 && Q + R <= 32);
        const uint32_t QR = Q + R;
        uint32_t logB = 0;
        while ((1u << logB) < QR) logB++;
        const uint32_t m = logB + logD;
        need(proof_len == 12 + 128 + 128ull * m + 96);
        const uint32_t hdr[3] = {logD, Q, R};
        tr_absorb_u32s(st, "relu/hdr", hdr, 3);
        F uZ[40], uA[40], uGA[40], uGZ[40], ub[72], cl[4], pt[72], fin[3];
        if (pts) {   // chained (D25): the points of the window's merged claims, nothing drawn
            for (uint32_t i = 0; i < logD; i++) {
                uZ[i] = ld(pts[i].b);
                uA[i] = ld(pts[logD + i].b);
                uGA[i] = ld(pts[2 * logD + i].b);
                uGZ[i] = ld(pts[3 * logD + i].b);
            }
        } else {
            for (uint32_t i = 0; i < logD; i++) uZ[i] = tr_challenge(st, "relu/uZ");
            for (uint32_t i = 0; i < logD; i++) uA[i] = tr_challenge(st, "relu/uA");
            for (uint32_t i = 0; i < logD; i++) uGA[i] = tr_challenge(st, "relu/uGA");
            for (uint32_t i = 0; i < logD; i++) uGZ[i] = tr_challenge(st, "relu/uGZ");
        }
        for (int i = 0; i < 4; i++) cl[i] = ld(proof + 12 + 32 * i);
        tr_absorb_frs(st, "relu/claims", cl, 4);
        const F r = tr_challenge(st, "relu/r"), rp = tr_challenge(st, "relu/rp");
        for (uint32_t i = 0; i < m; i++) ub[i] = tr_challenge(st, "relu/ubin");
        const F r2 = mul(r, r);
        // the combined claim r^2 Z~(u_Z) + r A~(u_A) + r'(r^2 G_A~(u_GA) + r G_Z~(u_GZ))
        F c = add(add(mul(r2, cl[0]), mul(r, cl[1])), mul(rp, add(mul(r2, cl[2]), mul(r, cl[3]))));
        const uint8_t* msgs = proof + 12 + 128;
        for (uint32_t t = 0; t < m; t++) {
            F ev[4];
            for (int X = 0; X < 4; X++) ev[X] = ld(msgs + 32ull * (4 * t + X));
            if (!eq(add(ev[0], ev[1]), c)) throw Reject{(int32_t)t + 1};
            tr_absorb_frs(st, "relu/msg", ev, 4);
            pt[t] = tr_challenge(st, "relu/x");
            c = interp(ev, 3, pt[t]);
        }
        for (int i = 0; i < 3; i++) fin[i] = ld(msgs + 128ull * m + 32 * i);
        const F* vj = pt;          // the j (bit position) variables are bound first (D2)
        const F* vi = pt + logB;
        // s(j) = 2^j (j < Q+R-1), -2^(Q+R-1) (j = Q+R-1): Z = sum_j s(j) bit_j (two's complement);
        // s'(j) = [j = R-1] + 2^(j-R) (R <= j < Q+R-1) - 2^(Q-1) [j = Q+R-1]: Z' = round(Z / 2^R)
        F s = zero(), sp = zero();
        for (uint32_t j = 0; j < QR; j++) {
            const F e = beta_at(vj, logB, j);
            const F sw = j == QR - 1 ? neg(from_u64(1ull << (QR - 1))) : from_u64(1ull << j);
            s = add(s, mul(e, sw));
            if (j + 1 >= R) {
                const F spw = j == R - 1 ? ONE : (j == QR - 1 ? neg(from_u64(1ull << (Q - 1))) : from_u64(1ull << (j - R)));
                sp = add(sp, mul(e, spw));
            }
        }
        const F bZ = beta(uZ, vi, logD), bA = beta(uA, vi, logD), bGA = beta(uGA, vi, logD), bGZ = beta(uGZ, vi, logD);
        const F bb = beta(ub, pt, m);
        const F a0 = fin[0], a1 = fin[1], oms = one_minus(fin[2]);
        F Pv = mul(r2, mul(bZ, mul(a0, s)));                                   // Z = sum_j s(j) bit_j
        Pv = add(Pv, mul(r, mul(bA, mul(oms, mul(a0, sp)))));                 // A = (1 - sigma) Z'
        Pv = add(Pv, mul(bb, sub(mul(a0, a0), a0)));                          // bits of Z are binary
        Pv = add(Pv, mul(mul(rp, r2), mul(bGA, mul(a1, s))));                 // G_A = sum_j s(j) bit_j
        Pv = add(Pv, mul(mul(rp, r), mul(bGZ, mul(oms, mul(a1, sp)))));       // G_Z = (1 - sigma) G_A'
        Pv = add(Pv, mul(rp, mul(bb, sub(mul(a1, a1), a1))));                 // bits of G_A are binary
        if (!eq(Pv, c)) throw Reject{-100};
        tr_absorb_frs(st, "relu/final", fin, 3);
        out_points(pt, m, point_out);
    });
}

// The loss-gradient family (Eq. fcnn-GZ-last, D24): the claims at the transcript's point u satisfy the
// linear identity G_Z~(u) = Z~(u) - Y~(u).
zk_status zk_verify_loss_grad(uint8_t st[32], uint32_t m, const zk_fr* claims, zk_fr* point_out, int32_t* fail) {
    return guarded(fail, [&] {
        need(st && claims && m >= 1 && m <= 64);
        tr_absorb_u32s(st, "lg/hdr", &m, 1);
        F u[64], cl[3];
        for (uint32_t t = 0; t < m; t++) u[t] = tr_challenge(st, "lg/u");
        for (int k = 0; k < 3; k++) cl[k] = ld(claims[k].b);
        if (!eq(cl[0], sub(cl[1], cl[2]))) throw Reject{-100};
        tr_absorb_frs(st, "lg/claims", cl, 3);
        out_points(u, m, point_out);
    });
}

// The zkReLU aux-claim merge (D21): rho, then the product sumcheck over (j, s) with n_eq = 0
// and the claim f0 + rho f1 + rho^2 f2 the verifier forms itself; the second final W~(r) is checked
// against the verifier's own evaluation of W, the first is the single merged claim aux~(r_s, v, r_j).
zk_status zk_verify_relu_merge(uint8_t st[32], uint32_t logD, uint32_t Q, uint32_t R, const zk_fr* relu_point,
                               const zk_fr* relu_finals, const uint8_t* proof, uint64_t proof_len, zk_fr* point_out,
                               int32_t* fail) {
    return guarded(fail, [&] {
        const uint32_t QR = Q + R;
        need(st && relu_point && relu_finals && proof && Q >= 1 && R >= 1 && Q <= 32 && R <= 32 && QR <= 32 && logD >= 1 && logD <= 40);
        uint32_t logB = 0;
        while ((1u << logB) < QR) logB++;
        const uint32_t m = logB + 1;
        need(proof_len == 12 + 32 + 32ull * m * 3 + 64 && rd32(proof) == m && rd32(proof + 4) == 0 && rd32(proof + 8) == 2);
        F w[8], f[3], r[8];
        for (uint32_t t = 0; t < logB; t++) w[t] = ld(relu_point[t].b);
        for (int k = 0; k < 3; k++) f[k] = ld(relu_finals[k].b);
        const F rho = tr_challenge(st, "relu/merge"), rho2 = mul(rho, rho);
        const F claim = add(add(f[0], mul(rho, f[1])), mul(rho2, f[2]));
        if (!eq(ld(proof + 12), claim)) throw Reject{-1};
        const uint32_t hdr[3] = {m, 0, 2};
        tr_absorb_u32s(st, "sc/hdr", hdr, 3);
        tr_absorb_frs(st, "sc/claim", &claim, 1);
        sumcheck_rounds(st, m, 0, 2, nullptr, claim, proof + 44, proof + 44 + 96ull * m, r);
        // W~(r_j, r_s) = (1 - r_s)(beta(w, r_j) + rho^2 eq(r_j, Q+R-1)) + r_s rho beta(w, r_j)
        const F bw = beta(w, r, logB), rs = r[logB];
        const F W = add(mul(one_minus(rs), add(bw, mul(rho2, beta_at(r, logB, QR - 1)))), mul(rs, mul(rho, bw)));
        if (!eq(ld(proof + 44 + 96ull * m + 32), W)) throw Reject{-101};
        out_points(r, m, point_out);
    });
}

// The claim merge (N3, D25; Eq. sc-reindex P:L262-270 in its general form): the verifier forms the
// phase-A claim sum_k rho_k c_k itself, recomputes P~(r_i, r_k) = sum_k beta(r_k, k) rho_k sum_j
// beta(u_k, j) beta(map_k[j], r_i) from the maps and Wy~(r_y) = sum_k beta(r_k, k) beta(v_k, r_y); the
// phase-B claim is phase A's second final.  Output: the stack point (r_y, r_i) and the claim X~ there.
zk_status zk_verify_claim_merge(uint8_t st[32], uint32_t n, uint32_t d, uint32_t K, const zk_cm_view* views,
                                const zk_fr* pts, const zk_fr* claims, const uint8_t* proof, uint64_t proof_len,
                                zk_fr* point_out, zk_fr* claim_out, int32_t* fail) {
    return guarded(fail, [&] {
        need(st && views && pts && claims && proof && K >= 1 && K <= 8 && n <= 16 && d >= 1 && d <= 40);
        uint32_t kap = 0;
        while ((1u << kap) < K) kap++;
        const uint32_t mA = n + kap;
        need(mA >= 1);
        const uint64_t la = 12 + 32 + 96ull * mA + 64, lb = 12 + 32 + 96ull * d + 64;
        need(proof_len == la + lb);
        if (rd32(proof) != mA || rd32(proof + 4) != 0 || rd32(proof + 8) != 2) throw Reject{-2};
        if (rd32(proof + la) != d || rd32(proof + la + 4) != 0 || rd32(proof + la + 8) != 2) throw Reject{-2};
        std::vector<uint32_t> hdr = {n, d, K};
        std::vector<F> cl(K), v(K * (size_t)d);
        std::vector<std::vector<F>> u(K);
        size_t po = 0;
        for (uint32_t k = 0; k < K; k++) {
            need(views[k].logN <= 16 && views[k].map);
            hdr.push_back(views[k].logN);
            cl[k] = ld(claims[k].b);
            for (uint32_t t = 0; t < d; t++) v[k * (size_t)d + t] = ld(pts[po++].b);
            for (uint32_t t = 0; t < views[k].logN; t++) u[k].push_back(ld(pts[po++].b));
            for (uint64_t j = 0; j < (1ull << views[k].logN); j++) {
                const uint32_t i = views[k].map[j];
                need(i == 0xffffffffu || (n < 32 && i < (1u << n)), ZK_ERR_RANGE);
            }
        }
        tr_absorb_u32s(st, "cm/hdr", hdr.data(), (uint32_t)hdr.size());
        tr_absorb_frs(st, "cm/claims", cl.data(), K);
        std::vector<F> rho(K);
        F cA = zero();
        for (uint32_t k = 0; k < K; k++) {
            rho[k] = tr_challenge(st, "cm/rho");
            cA = add(cA, mul(rho[k], cl[k]));
        }
        if (!eq(ld(proof + 12), cA)) throw Reject{-1};
        const uint32_t hA[3] = {mA, 0, 2};
        tr_absorb_u32s(st, "sc/hdr", hA, 3);
        tr_absorb_frs(st, "sc/claim", &cA, 1);
        F rA[64], rB[64];
        sumcheck_rounds(st, mA, 0, 2, nullptr, cA, proof + 44, proof + 44 + 96ull * mA, rA);
        const F* ri = rA;
        const F* rk = rA + n;
        F Pv = zero();
        for (uint32_t k = 0; k < K; k++) {
            F sk = zero();
            for (uint64_t j = 0; j < (1ull << views[k].logN); j++) {
                const uint32_t i = views[k].map[j];
                if (i == 0xffffffffu) continue;
                sk = add(sk, mul(beta_at(u[k].data(), views[k].logN, j), beta_at(ri, n, i)));
            }
            Pv = add(Pv, mul(beta_at(rk, kap, k), mul(rho[k], sk)));
        }
        if (!eq(ld(proof + 44 + 96ull * mA), Pv)) throw Reject{-101};
        const F cB = ld(proof + 44 + 96ull * mA + 32);
        const uint8_t* pb = proof + la;
        if (!eq(ld(pb + 12), cB)) throw Reject{-1};
        const uint32_t hB[3] = {d, 0, 2};
        tr_absorb_u32s(st, "sc/hdr", hB, 3);
        tr_absorb_frs(st, "sc/claim", &cB, 1);
        sumcheck_rounds(st, d, 0, 2, nullptr, cB, pb + 44, pb + 44 + 96ull * d, rB);
        F Wv = zero();
        for (uint32_t k = 0; k < K; k++) Wv = add(Wv, mul(beta_at(rk, kap, k), beta(&v[k * (size_t)d], rB, d)));
        if (!eq(ld(pb + 44 + 96ull * d), Wv)) throw Reject{-102};
        out_points(rB, d, point_out);
        if (point_out) out_points(ri, n, point_out + d);
        if (claim_out) store(ld(pb + 44 + 96ull * d + 32), claim_out->b);
    });
}

// The top-layer rescale (D26): A from the claim r Z~(u_Z) + Z'~(u_P) with the weight final recomputed from
// the verifier's own beta, s and s' evaluations; B from 0 in the eq form (Protocol 3) with its second
// final = the first minus one (the MLE of aux - 1).
zk_status zk_verify_rescale(uint8_t st[32], const uint8_t* proof, uint64_t proof_len, const uint32_t expect[3],
                            const zk_fr* pts, zk_fr* claims_out, zk_fr* aux_out, zk_fr* point_out, int32_t* fail) {
    return guarded(fail, [&] {
        need(st && proof && expect && pts && proof_len >= 12);
        const uint32_t logD = rd32(proof), Q = rd32(proof + 4), R = rd32(proof + 8);
        if (logD != expect[0] || Q != expect[1] || R != expect[2]) throw Reject{-2};
        need(logD >= 1 && logD <= 40 && Q >= 1 && R >= 1 && Q <= 32 && R <= 32 && Q + R <= 32);
        const uint32_t QR = Q + R;
        uint32_t logB = 0;
        while ((1u << logB) < QR) logB++;
        const uint32_t m = logB + logD;
        const uint64_t lp = 12 + 32 + 96ull * m + 64;
        need(proof_len == 12 + 64 + 2 * lp);
        const uint8_t *pa = proof + 76, *pb = proof + 76 + lp;
        if (rd32(pa) != m || rd32(pa + 4) != 0 || rd32(pa + 8) != 2) throw Reject{-2};
        if (rd32(pb) != m || rd32(pb + 4) != m || rd32(pb + 8) != 2) throw Reject{-2};
        const uint32_t hdr[3] = {logD, Q, R};
        tr_absorb_u32s(st, "rs/hdr", hdr, 3);
        F uZ[40], uP[40], cl[2];
        for (uint32_t i = 0; i < logD; i++) {
            uZ[i] = ld(pts[i].b);
            uP[i] = ld(pts[logD + i].b);
        }
        cl[0] = ld(proof + 12);
        cl[1] = ld(proof + 44);
        tr_absorb_frs(st, "rs/claims", cl, 2);
        const F r = tr_challenge(st, "rs/r");
        const F cA = add(mul(r, cl[0]), cl[1]);
        if (!eq(ld(pa + 12), cA)) throw Reject{-1};
        const uint32_t hA[3] = {m, 0, 2};
        tr_absorb_u32s(st, "sc/hdr", hA, 3);
        tr_absorb_frs(st, "sc/claim", &cA, 1);
        F rA[80], rB[80], w[80];
        sumcheck_rounds(st, m, 0, 2, nullptr, cA, pa + 44, pa + 44 + 96ull * m, rA);
        const F* vj = rA;
        const F* vi = rA + logB;
        F sv = zero(), spv = zero();
        for (uint32_t j = 0; j < QR; j++) {
            const F e = beta_at(vj, logB, j);
            sv = add(sv, mul(e, j == QR - 1 ? neg(from_u64(1ull << (QR - 1))) : from_u64(1ull << j)));
            if (j + 1 >= R) {
                const F spw = j == R - 1 ? ONE : (j == QR - 1 ? neg(from_u64(1ull << (Q - 1))) : from_u64(1ull << (j - R)));
                spv = add(spv, mul(e, spw));
            }
        }
        const F Wv = add(mul(r, mul(beta(uZ, vi, logD), sv)), mul(beta(uP, vi, logD), spv));
        if (!eq(ld(pa + 44 + 96ull * m), Wv)) throw Reject{-101};
        for (uint32_t t = 0; t < m; t++) w[t] = tr_challenge(st, "rs/w");
        if (!eq(ld(pb + 12), zero())) throw Reject{-1};
        const uint32_t hB[3] = {m, m, 2};
        tr_absorb_u32s(st, "sc/hdr", hB, 3);
        const F z = zero();
        tr_absorb_frs(st, "sc/claim", &z, 1);
        sumcheck_rounds(st, m, m, 2, w, z, pb + 44, pb + 44 + 96ull * m, rB);
        const F b0 = ld(pb + 44 + 96ull * m), b1 = ld(pb + 44 + 96ull * m + 32);
        if (!eq(b1, sub(b0, ONE))) throw Reject{-102};
        if (claims_out) {
            store(cl[0], claims_out[0].b);
            store(cl[1], claims_out[1].b);
        }
        if (aux_out) {
            store(ld(pa + 44 + 96ull * m + 32), aux_out[0].b);
            store(b0, aux_out[1].b);
        }
        out_points(rA, m, point_out);
        if (point_out) out_points(rB, m, point_out + m);
    });
}

}  // extern "C"
