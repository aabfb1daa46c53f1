// fr64.cuh — the Fr Montgomery product on the FP64 pipe (DESIGN.md §6 "Fr product").
//
// Same function as fr_mul (fr.cuh): a * b * 2^-256 mod p on the 8 x 32-bit Montgomery representation,
// bit for bit.  The 64 32-bit half-products of the integer CIOS run on the IMAD (fmaheavy) pipe, where
// IMAD.WIDE costs two issue slots: ~376 slots per product, 48.9 G/s measured.  The B200's FP64 pipe
// (DFMA at 64 lanes/SM/clk, idle otherwise) computes a 52 x 52 -> 104-bit product exactly in two fused
// multiply-adds (the split of Emmart, Zheng & Weems, ARITH 2018):
//     h = fma_rz(x, y, 2^104)                  = 2^104 + floor(xy / 2^52) 2^52    (bits: 0x467.. + hi)
//     l = fma_rz(x, y, (2^104 + 2^52) - h)     = 2^52 + (xy mod 2^52)              (bits: 0x433.. + lo)
// so with 52-bit limbs (5 per element) the product is 25 such pairs, and the raw bit patterns are summed
// as 64-bit integers into column accumulators (the exponent biases are multiples of 2^52: they vanish
// mod 2^52 and are pre-subtracted once per column, so no per-term masking).  Montgomery reduction
// with word 2^52 and R' = 2^260: q_i = (c_i * (-p^-1)) mod 2^52 by the same split (its low half only),
// then 5 more pairs q_i p_j.  Because R' = 2^4 R, the first operand enters as 16 a (a < p, so 16 a b <
// p R' and the result is < 2p: one conditional subtraction), which gives exactly a b R^-1.
// Per product: 185 FP64-pipe operations (DFMA/DADD) and ~200 ALU operations (limb extraction, 64-bit
// column sums), against ~376 fmaheavy slots for the integer CIOS.
#pragma once
// included by fr.cuh after fr_t and fr_reduce_once

namespace zk {

#define ZK_F52_MASK 0x000fffffffffffffull
#define ZK_F52_EXP 0x4330000000000000ull   // bits of 2^52
#define ZK_TWO52 4503599627370496.0                           // 2^52
#define ZK_TWO104 20282409603651670423947251286016.0           // 2^104
#define ZK_C2 20282409603651674927546878656512.0               // 2^104 + 2^52

__device__ __forceinline__ double zk_f64(uint64_t b) { return __longlong_as_double((long long)b); }
__device__ __forceinline__ uint64_t zk_bits(double d) { return (uint64_t)__double_as_longlong(d); }

// bits [lo, lo + 52) of the 256-bit integer a (lo may be negative: zero-filled), as an exact double
__device__ __forceinline__ double fr64_limb(const fr_t& a, int lo) {
    uint64_t x;
    if (lo < 0) {
        x = ((uint64_t)a.v[0] | ((uint64_t)a.v[1] << 32)) << (-lo);
    } else {
        const int w = lo >> 5, o = lo & 31;
        const uint64_t w0 = a.v[w], w1 = w + 1 < 8 ? a.v[w + 1] : 0u, w2 = w + 2 < 8 ? a.v[w + 2] : 0u;
        x = (w0 | (w1 << 32)) >> o;
        if (o > 12) x |= w2 << (64 - o);
    }
    return __dsub_rn(zk_f64((x & ZK_F52_MASK) | ZK_F52_EXP), ZK_TWO52);
}

// clo += low 52 bits of x*y (as a biased pattern), chi += high part (biased pattern)
#define ZK_F64_MAC(x, y, clo, chi)                                                                     \
    do {                                                                                               \
        const double h_ = __fma_rz((x), (y), ZK_TWO104);                                               \
        const double l_ = __fma_rz((x), (y), __dsub_rn(ZK_C2, h_));                                    \
        (clo) += zk_bits(l_);                                                                          \
        (chi) += zk_bits(h_);                                                                          \
    } while (0)

__device__ __forceinline__ fr_t fr_mul_f64(const fr_t& a, const fr_t& b) {
    // p in 52-bit limbs, -p^-1 mod 2^52
    const double P0 = 4503595332403201.0, P1 = 52776117727231.0, P2 = 2711223964777892.0,
                 P3 = 2203984808738944.0, P4 = 127464551688605.0;   // limbs of p (tests/test_build.py re-derives them)
    const double PINV = 4503595332403199.0;
    const double A[5] = {fr64_limb(a, -4), fr64_limb(a, 48), fr64_limb(a, 100), fr64_limb(a, 152), fr64_limb(a, 204)};
    const double B[5] = {fr64_limb(b, 0), fr64_limb(b, 52), fr64_limb(b, 104), fr64_limb(b, 156), fr64_limb(b, 208)};
    // column accumulators, pre-biased by minus every exponent pattern they will receive
    uint64_t c[10] = {0x79a0000000000000ull, 0x6660000000000000ull, 0x5320000000000000ull, 0x3fe0000000000000ull,
                      0x2ca0000000000000ull, 0x2620000000000000ull, 0x3960000000000000ull, 0x4ca0000000000000ull,
                      0x5fe0000000000000ull, 0x7320000000000000ull};
#pragma unroll
    for (int i = 0; i < 5; i++)
#pragma unroll
        for (int j = 0; j < 5; j++) ZK_F64_MAC(A[i], B[j], c[i + j], c[i + j + 1]);
    const double Pl[5] = {P0, P1, P2, P3, P4};
#pragma unroll
    for (int i = 0; i < 5; i++) {
        const double x = __dsub_rn(zk_f64((c[i] & ZK_F52_MASK) | ZK_F52_EXP), ZK_TWO52);
        const double h = __fma_rz(x, PINV, ZK_TWO104);
        const double q = __dsub_rn(__fma_rz(x, PINV, __dsub_rn(ZK_C2, h)), ZK_TWO52);   // (x * PINV) mod 2^52
#pragma unroll
        for (int j = 0; j < 5; j++) ZK_F64_MAC(q, Pl[j], c[i + j], c[i + j + 1]);
        c[i + 1] += c[i] >> 52;   // c[i] = 0 mod 2^52 now, and exact
    }
#pragma unroll
    for (int k = 5; k < 9; k++) {
        c[k + 1] += c[k] >> 52;
        c[k] &= ZK_F52_MASK;
    }
    const uint64_t u0 = c[5] | (c[6] << 52), u1 = (c[6] >> 12) | (c[7] << 40), u2 = (c[7] >> 24) | (c[8] << 28),
                   u3 = (c[8] >> 36) | (c[9] << 16);
    fr_t r;
    r.v[0] = (uint32_t)u0; r.v[1] = (uint32_t)(u0 >> 32);
    r.v[2] = (uint32_t)u1; r.v[3] = (uint32_t)(u1 >> 32);
    r.v[4] = (uint32_t)u2; r.v[5] = (uint32_t)(u2 >> 32);
    r.v[6] = (uint32_t)u3; r.v[7] = (uint32_t)(u3 >> 32);
    return fr_reduce_once(r);
}

// The same product with the reduction interleaved row by row (CIOS order) in a rolled loop: the six live
// columns shift down one limb per row (the column entering at the top starts at its pre-bias, which the
// constants above give: 0x3960.. + i 0x1340.. for columns 6..9), and A's limbs shift with them, so every
// index is static and the body is ~5x smaller (~1.8 KB against ~7 KB: inside the L0 instruction cache).
// Every column receives the same terms as in fr_mul_f64, so the result is the same bits.
__device__ __forceinline__ fr_t fr_mul_f64r(const fr_t& a, const fr_t& b) {
    const double P0 = 4503595332403201.0, P1 = 52776117727231.0, P2 = 2711223964777892.0,
                 P3 = 2203984808738944.0, P4 = 127464551688605.0;
    const double PINV = 4503595332403199.0;
    double A[5] = {fr64_limb(a, -4), fr64_limb(a, 48), fr64_limb(a, 100), fr64_limb(a, 152), fr64_limb(a, 204)};
    const double B[5] = {fr64_limb(b, 0), fr64_limb(b, 52), fr64_limb(b, 104), fr64_limb(b, 156), fr64_limb(b, 208)};
    const double Pl[5] = {P0, P1, P2, P3, P4};
    uint64_t c[6] = {0x79a0000000000000ull, 0x6660000000000000ull, 0x5320000000000000ull, 0x3fe0000000000000ull,
                     0x2ca0000000000000ull, 0x2620000000000000ull};
#pragma unroll 1
    for (int i = 0; i < 5; i++) {
        const double ai = A[0];
#pragma unroll
        for (int j = 0; j < 5; j++) ZK_F64_MAC(ai, B[j], c[j], c[j + 1]);
        const double x = __dsub_rn(zk_f64((c[0] & ZK_F52_MASK) | ZK_F52_EXP), ZK_TWO52);
        const double h = __fma_rz(x, PINV, ZK_TWO104);
        const double q = __dsub_rn(__fma_rz(x, PINV, __dsub_rn(ZK_C2, h)), ZK_TWO52);
#pragma unroll
        for (int j = 0; j < 5; j++) ZK_F64_MAC(q, Pl[j], c[j], c[j + 1]);
        const uint64_t carry = c[0] >> 52;
        c[0] = c[1] + carry;
        c[1] = c[2];
        c[2] = c[3];
        c[3] = c[4];
        c[4] = c[5];
        c[5] = i < 4 ? 0x3960000000000000ull + (uint64_t)i * 0x1340000000000000ull : 0ull;
        A[0] = A[1];
        A[1] = A[2];
        A[2] = A[3];
        A[3] = A[4];
    }
#pragma unroll
    for (int k = 0; k < 4; k++) {
        c[k + 1] += c[k] >> 52;
        c[k] &= ZK_F52_MASK;
    }
    const uint64_t u0 = c[0] | (c[1] << 52), u1 = (c[1] >> 12) | (c[2] << 40), u2 = (c[2] >> 24) | (c[3] << 28),
                   u3 = (c[3] >> 36) | (c[4] << 16);
    fr_t r;
    r.v[0] = (uint32_t)u0; r.v[1] = (uint32_t)(u0 >> 32);
    r.v[2] = (uint32_t)u1; r.v[3] = (uint32_t)(u1 >> 32);
    r.v[4] = (uint32_t)u2; r.v[5] = (uint32_t)(u2 >> 32);
    r.v[6] = (uint32_t)u3; r.v[7] = (uint32_t)(u3 >> 32);
    return fr_reduce_once(r);
}

}  // namespace zk
