// fr.cuh — BLS12-381 scalar field Fr on sm_100a (D1).
//
// Representation: 8 x 32-bit little-endian limbs, Montgomery form with R = 2^256,
// array-of-structs in HBM (32 B per element, two 16-B vector accesses).
// Multiplication: CIOS (coarsely integrated operand scanning) with PTX carry
// chains: per limb b_i one mad.lo chain and one mad.hi chain for a*b_i, then
// m = t_0 * n0 (n0 = -p^{-1} mod 2^32 = 0xffffffff) and the same two chains for
// m*p.  Because p < 2^255 the running value stays < 2p and every pre-shift sum
// < 2p * 2^32 < 2^288, so 9 limbs suffice (no carry word).  Constants below were
// derived with Python integers (tests/test_build.py re-derives them).
#pragma once
#include <stdint.h>

namespace zk {

struct __align__(16) fr_t { uint32_t v[8]; };

// p = 0x73eda753299d7d483339d80809a1d80553bda402fffe5bfeffffffff00000001
#define ZK_P0 0x00000001u
#define ZK_P1 0xffffffffu
#define ZK_P2 0xfffe5bfeu
#define ZK_P3 0x53bda402u
#define ZK_P4 0x09a1d805u
#define ZK_P5 0x3339d808u
#define ZK_P6 0x299d7d48u
#define ZK_P7 0x73eda753u

__host__ __device__ constexpr fr_t fr_const(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                            uint32_t a4, uint32_t a5, uint32_t a6, uint32_t a7) {
    return fr_t{{a0, a1, a2, a3, a4, a5, a6, a7}};
}
// R mod p (Montgomery 1), R^2 mod p, R^3 mod p, Montgomery form of 2^31
#define ZK_ONE  fr_const(0xfffffffeu, 0x00000001u, 0x00034802u, 0x5884b7fau, 0xecbc4ff5u, 0x998c4fefu, 0xacc5056fu, 0x1824b159u)
#define ZK_R2   fr_const(0xf3f29c6du, 0xc999e990u, 0x87925c23u, 0x2b6cedcbu, 0x7254398fu, 0x05d31496u, 0x9f59ff11u, 0x0748d9d9u)
#define ZK_R3   fr_const(0x439b73afu, 0xc62c1807u, 0x8cf06990u, 0x1b3e0d18u, 0xc7b5f418u, 0x73d13c71u, 0xc8db33e9u, 0x6e2a5bb9u)
#define ZK_TWO31_MONT fr_const(0xe557b58au, 0x1aa84a74u, 0x34d1e277u, 0xa537585bu, 0x25370837u, 0x0b017f57u, 0x8b620bfbu, 0x73ac0a47u)

__device__ __forceinline__ fr_t fr_zero() { return fr_t{{0, 0, 0, 0, 0, 0, 0, 0}}; }
__device__ __forceinline__ fr_t fr_one() { return ZK_ONE; }

__device__ __forceinline__ bool fr_is_zero(const fr_t& a) {
    return (a.v[0] | a.v[1] | a.v[2] | a.v[3] | a.v[4] | a.v[5] | a.v[6] | a.v[7]) == 0;
}
__device__ __forceinline__ bool fr_equal(const fr_t& a, const fr_t& b) {
    uint32_t d = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) d |= a.v[i] ^ b.v[i];
    return d == 0;
}

// x - p if x >= p (x < 2p < 2^256), branch-free
__device__ __forceinline__ fr_t fr_reduce_once(const fr_t& x) {
    fr_t r;
    uint32_t borrow;
    asm("sub.cc.u32  %0, %9,  %17;\n\t"
        "subc.cc.u32 %1, %10, %18;\n\t"
        "subc.cc.u32 %2, %11, %19;\n\t"
        "subc.cc.u32 %3, %12, %20;\n\t"
        "subc.cc.u32 %4, %13, %21;\n\t"
        "subc.cc.u32 %5, %14, %22;\n\t"
        "subc.cc.u32 %6, %15, %23;\n\t"
        "subc.cc.u32 %7, %16, %24;\n\t"
        "subc.u32    %8, 0, 0;"
        : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]), "=r"(r.v[6]),
          "=r"(r.v[7]), "=r"(borrow)
        : "r"(x.v[0]), "r"(x.v[1]), "r"(x.v[2]), "r"(x.v[3]), "r"(x.v[4]), "r"(x.v[5]), "r"(x.v[6]), "r"(x.v[7]),
          "n"(ZK_P0), "n"(ZK_P1), "n"(ZK_P2), "n"(ZK_P3), "n"(ZK_P4), "n"(ZK_P5), "n"(ZK_P6), "n"(ZK_P7));
    // borrow = 0xffffffff when x < p: keep x
#pragma unroll
    for (int i = 0; i < 8; i++) r.v[i] = borrow ? x.v[i] : r.v[i];
    return r;
}

__device__ __forceinline__ fr_t fr_add(const fr_t& a, const fr_t& b) {
    fr_t s;
    asm("add.cc.u32  %0, %8,  %16;\n\t"
        "addc.cc.u32 %1, %9,  %17;\n\t"
        "addc.cc.u32 %2, %10, %18;\n\t"
        "addc.cc.u32 %3, %11, %19;\n\t"
        "addc.cc.u32 %4, %12, %20;\n\t"
        "addc.cc.u32 %5, %13, %21;\n\t"
        "addc.cc.u32 %6, %14, %22;\n\t"
        "addc.u32    %7, %15, %23;"
        : "=r"(s.v[0]), "=r"(s.v[1]), "=r"(s.v[2]), "=r"(s.v[3]), "=r"(s.v[4]), "=r"(s.v[5]), "=r"(s.v[6]), "=r"(s.v[7])
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]),
          "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    return fr_reduce_once(s);   // a + b < 2p < 2^256: no carry out
}

__device__ __forceinline__ fr_t fr_sub(const fr_t& a, const fr_t& b) {
    fr_t d;
    uint32_t borrow;
    asm("sub.cc.u32  %0, %9,  %17;\n\t"
        "subc.cc.u32 %1, %10, %18;\n\t"
        "subc.cc.u32 %2, %11, %19;\n\t"
        "subc.cc.u32 %3, %12, %20;\n\t"
        "subc.cc.u32 %4, %13, %21;\n\t"
        "subc.cc.u32 %5, %14, %22;\n\t"
        "subc.cc.u32 %6, %15, %23;\n\t"
        "subc.cc.u32 %7, %16, %24;\n\t"
        "subc.u32    %8, 0, 0;"
        : "=r"(d.v[0]), "=r"(d.v[1]), "=r"(d.v[2]), "=r"(d.v[3]), "=r"(d.v[4]), "=r"(d.v[5]), "=r"(d.v[6]),
          "=r"(d.v[7]), "=r"(borrow)
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]),
          "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    // add (p & borrow)
    const uint32_t m = borrow;
    asm("add.cc.u32  %0, %0, %8;\n\t"
        "addc.cc.u32 %1, %1, %9;\n\t"
        "addc.cc.u32 %2, %2, %10;\n\t"
        "addc.cc.u32 %3, %3, %11;\n\t"
        "addc.cc.u32 %4, %4, %12;\n\t"
        "addc.cc.u32 %5, %5, %13;\n\t"
        "addc.cc.u32 %6, %6, %14;\n\t"
        "addc.u32    %7, %7, %15;"
        : "+r"(d.v[0]), "+r"(d.v[1]), "+r"(d.v[2]), "+r"(d.v[3]), "+r"(d.v[4]), "+r"(d.v[5]), "+r"(d.v[6]), "+r"(d.v[7])
        : "r"(ZK_P0 & m), "r"(ZK_P1 & m), "r"(ZK_P2 & m), "r"(ZK_P3 & m), "r"(ZK_P4 & m), "r"(ZK_P5 & m),
          "r"(ZK_P6 & m), "r"(ZK_P7 & m));
    return d;
}

__device__ __forceinline__ fr_t fr_neg(const fr_t& a) { return fr_sub(fr_zero(), a); }
__device__ __forceinline__ fr_t fr_dbl(const fr_t& a) { return fr_add(a, a); }

// t[0..8] += a[0..7] * bi   (two carry chains; total stays < 2^288 by the CIOS bound)
#define ZK_MAC_ROW(t, a, bi)                                                                           \
    asm("mad.lo.cc.u32  %0, %9,  %17, %0;\n\t"                                                         \
        "madc.lo.cc.u32 %1, %10, %17, %1;\n\t"                                                         \
        "madc.lo.cc.u32 %2, %11, %17, %2;\n\t"                                                         \
        "madc.lo.cc.u32 %3, %12, %17, %3;\n\t"                                                         \
        "madc.lo.cc.u32 %4, %13, %17, %4;\n\t"                                                         \
        "madc.lo.cc.u32 %5, %14, %17, %5;\n\t"                                                         \
        "madc.lo.cc.u32 %6, %15, %17, %6;\n\t"                                                         \
        "madc.lo.cc.u32 %7, %16, %17, %7;\n\t"                                                         \
        "addc.u32       %8, %8, 0;\n\t"                                                                \
        "mad.hi.cc.u32  %1, %9,  %17, %1;\n\t"                                                         \
        "madc.hi.cc.u32 %2, %10, %17, %2;\n\t"                                                         \
        "madc.hi.cc.u32 %3, %11, %17, %3;\n\t"                                                         \
        "madc.hi.cc.u32 %4, %12, %17, %4;\n\t"                                                         \
        "madc.hi.cc.u32 %5, %13, %17, %5;\n\t"                                                         \
        "madc.hi.cc.u32 %6, %14, %17, %6;\n\t"                                                         \
        "madc.hi.cc.u32 %7, %15, %17, %7;\n\t"                                                         \
        "madc.hi.u32    %8, %16, %17, %8;"                                                             \
        : "+r"(t[0]), "+r"(t[1]), "+r"(t[2]), "+r"(t[3]), "+r"(t[4]), "+r"(t[5]), "+r"(t[6]), "+r"(t[7]), \
          "+r"(t[8])                                                                                   \
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]), "r"(bi))

// t[0..8] += p * m, then t >>= 32 (t[0] becomes 0 by construction of m)
#define ZK_REDC_ROW(t)                                                                                 \
    do {                                                                                               \
        uint32_t m_ = t[0] * 0xffffffffu;                                                              \
        asm("mad.lo.cc.u32  %0, %9, %10, %0;\n\t"                                                      \
            "madc.lo.cc.u32 %1, %9, %11, %1;\n\t"                                                      \
            "madc.lo.cc.u32 %2, %9, %12, %2;\n\t"                                                      \
            "madc.lo.cc.u32 %3, %9, %13, %3;\n\t"                                                      \
            "madc.lo.cc.u32 %4, %9, %14, %4;\n\t"                                                      \
            "madc.lo.cc.u32 %5, %9, %15, %5;\n\t"                                                      \
            "madc.lo.cc.u32 %6, %9, %16, %6;\n\t"                                                      \
            "madc.lo.cc.u32 %7, %9, %17, %7;\n\t"                                                      \
            "addc.u32       %8, %8, 0;\n\t"                                                            \
            "mad.hi.cc.u32  %1, %9, %10, %1;\n\t"                                                      \
            "madc.hi.cc.u32 %2, %9, %11, %2;\n\t"                                                      \
            "madc.hi.cc.u32 %3, %9, %12, %3;\n\t"                                                      \
            "madc.hi.cc.u32 %4, %9, %13, %4;\n\t"                                                      \
            "madc.hi.cc.u32 %5, %9, %14, %5;\n\t"                                                      \
            "madc.hi.cc.u32 %6, %9, %15, %6;\n\t"                                                      \
            "madc.hi.cc.u32 %7, %9, %16, %7;\n\t"                                                      \
            "madc.hi.u32    %8, %9, %17, %8;"                                                          \
            : "+r"(t[0]), "+r"(t[1]), "+r"(t[2]), "+r"(t[3]), "+r"(t[4]), "+r"(t[5]), "+r"(t[6]),    \
              "+r"(t[7]), "+r"(t[8])                                                                   \
            : "r"(m_), "n"(ZK_P0), "n"(ZK_P1), "n"(ZK_P2), "n"(ZK_P3), "n"(ZK_P4), "n"(ZK_P5),        \
              "n"(ZK_P6), "n"(ZK_P7));                                                                 \
        t[0] = t[1]; t[1] = t[2]; t[2] = t[3]; t[3] = t[4]; t[4] = t[5]; t[5] = t[6]; t[6] = t[7];     \
        t[7] = t[8]; t[8] = 0;                                                                         \
    } while (0)

// Montgomery product a * b * R^{-1} mod p.  Requires a < p; b may be any value < 2^256.
// CIOS with 64-bit intermediates left to the compiler (IMAD.WIDE.U32 + IADD3 carries it schedules
// freely across independent products — 23% faster than hand-written PTX carry chains on the B200,
// scripts/mulbench.cu), using p0 = 1 (m p0 + t0 = 0 mod 2^32, carry t0 != 0) and p1 = 2^32 - 1
// (m p1 = (m << 32) - m on the ALU pipe, relieving the FMA pipe).
__device__ __forceinline__ fr_t fr_mul(const fr_t& a, const fr_t& b) {
    const uint32_t p[8] = {ZK_P0, ZK_P1, ZK_P2, ZK_P3, ZK_P4, ZK_P5, ZK_P6, ZK_P7};
    uint32_t t[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint64_t C = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint64_t uv = (uint64_t)a.v[j] * b.v[i] + t[j] + C;
            t[j] = (uint32_t)uv;
            C = uv >> 32;
        }
        t[8] += (uint32_t)C;
        const uint32_t m = t[0] * 0xffffffffu;   // = -t0 mod 2^32
        C = (uint64_t)(t[0] != 0);
        {
            const uint64_t uv = ((uint64_t)m << 32) + t[1] + C - m;
            t[0] = (uint32_t)uv;
            C = uv >> 32;
        }
#pragma unroll
        for (int j = 2; j < 8; j++) {
            const uint64_t uv = (uint64_t)m * p[j] + t[j] + C;
            t[j - 1] = (uint32_t)uv;
            C = uv >> 32;
        }
        const uint64_t uv = (uint64_t)t[8] + C;
        t[7] = (uint32_t)uv;
        t[8] = (uint32_t)(uv >> 32);
    }
    fr_t r;
#pragma unroll
    for (int i = 0; i < 8; i++) r.v[i] = t[i];
    return fr_reduce_once(r);
}
__device__ __forceinline__ fr_t fr_sqr(const fr_t& a) { return fr_mul(a, a); }

}  // namespace zk
#include "fr64.cuh"
namespace zk {

// The product of the hot out-of-line bodies below: the FP64-pipe product (fr64.cuh) unless the build
// selects the integer CIOS (ZKDL_FR64=0); both give identical bits.
#ifndef ZKDL_FR64
#define ZKDL_FR64 1
#endif
__device__ __forceinline__ fr_t fr_mul_hot(const fr_t& a, const fr_t& b) {
#if ZKDL_FR64 == 2
    return fr_mul_f64r(a, b);   // the rolled (CIOS-order) FP64 product: a ~5x smaller body
#elif ZKDL_FR64
    return fr_mul_f64(a, b);
#else
    return fr_mul(a, b);
#endif
}

// Out-of-line but fully unrolled product for hot loops with many multiplications: one ~560-instruction
// body shared by every call site keeps the loop inside the instruction cache (the inlined k_relu_iround
// body was > 100 KB of SASS; ncu stall_no_inst 36%).
static __device__ __noinline__ fr_t fr_mul_ni(fr_t a, fr_t b) { return fr_mul_hot(a, b); }

// Three independent products in one out-of-line body: the scheduler interleaves the three CIOS
// chains, so a warp has three-way instruction-level parallelism inside the product (the single
// product is a dependent chain that leaves the pipes idle at low occupancy).
struct fr3_t { fr_t x, y, z; };
static __device__ __noinline__ fr3_t fr_mul3_ni(fr_t a0, fr_t b0, fr_t a1, fr_t b1, fr_t a2, fr_t b2) {
    return fr3_t{fr_mul_hot(a0, b0), fr_mul_hot(a1, b1), fr_mul_hot(a2, b2)};
}

// Two independent products in one out-of-line body (for the groups with only two products: a wasted
// third slot of fr_mul3_ni costs a whole product)
struct fr2p_t { fr_t x, y; };
static __device__ __noinline__ fr2p_t fr_mul2_ni(fr_t a0, fr_t b0, fr_t a1, fr_t b1) {
    return fr2p_t{fr_mul_hot(a0, b0), fr_mul_hot(a1, b1)};
}

// One out-of-line copy for cold code (finalizers, single-CTA round kernels): the inlined product is
// ~560 SASS instructions, and cold code that inlines dozens of them runs out of the instruction
// cache (ncu: stall_no_inst dominated the round kernels' finalize).
static __device__ __noinline__ fr_t fr_mul_cold(fr_t a, fr_t b) {
    // rolled over the 8 limbs of b (one MAC row + one REDC row of code, ~10x smaller than fr_mul)
    uint32_t t[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t bb[8] = {b.v[0], b.v[1], b.v[2], b.v[3], b.v[4], b.v[5], b.v[6], b.v[7]};
#pragma unroll 1
    for (int i = 0; i < 8; i++) {
        const uint32_t bi = bb[0];
        bb[0] = bb[1]; bb[1] = bb[2]; bb[2] = bb[3]; bb[3] = bb[4]; bb[4] = bb[5]; bb[5] = bb[6]; bb[6] = bb[7];
        ZK_MAC_ROW(t, a.v, bi);
        ZK_REDC_ROW(t);
    }
    fr_t r;
#pragma unroll
    for (int i = 0; i < 8; i++) r.v[i] = t[i];
    return fr_reduce_once(r);
}

// Montgomery reduction of a wide unsigned integer T (10 limbs, T < p * 2^256):
// returns T * R^{-1} mod p.  Used by the int32 x Fr lazy accumulators.
__device__ __forceinline__ fr_t fr_redc_wide(const uint32_t w[10]) {
    uint32_t t[9] = {w[0], w[1], w[2], w[3], w[4], w[5], w[6], w[7], w[8]};
    uint32_t hi = w[9];
    // 8 reduction steps; after each shift the next input limb enters at t[8]
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint32_t m_ = t[0] * 0xffffffffu;
        uint32_t carry;
        asm("mad.lo.cc.u32  %0, %10, %11, %0;\n\t"
            "madc.lo.cc.u32 %1, %10, %12, %1;\n\t"
            "madc.lo.cc.u32 %2, %10, %13, %2;\n\t"
            "madc.lo.cc.u32 %3, %10, %14, %3;\n\t"
            "madc.lo.cc.u32 %4, %10, %15, %4;\n\t"
            "madc.lo.cc.u32 %5, %10, %16, %5;\n\t"
            "madc.lo.cc.u32 %6, %10, %17, %6;\n\t"
            "madc.lo.cc.u32 %7, %10, %18, %7;\n\t"
            "addc.cc.u32    %8, %8, 0;\n\t"
            "addc.u32       %9, 0, 0;\n\t"
            "mad.hi.cc.u32  %1, %10, %11, %1;\n\t"
            "madc.hi.cc.u32 %2, %10, %12, %2;\n\t"
            "madc.hi.cc.u32 %3, %10, %13, %3;\n\t"
            "madc.hi.cc.u32 %4, %10, %14, %4;\n\t"
            "madc.hi.cc.u32 %5, %10, %15, %5;\n\t"
            "madc.hi.cc.u32 %6, %10, %16, %6;\n\t"
            "madc.hi.cc.u32 %7, %10, %17, %7;\n\t"
            "madc.hi.cc.u32 %8, %10, %18, %8;\n\t"
            "addc.u32       %9, %9, 0;"
            : "+r"(t[0]), "+r"(t[1]), "+r"(t[2]), "+r"(t[3]), "+r"(t[4]), "+r"(t[5]), "+r"(t[6]), "+r"(t[7]),
              "+r"(t[8]), "=r"(carry)
            : "r"(m_), "n"(ZK_P0), "n"(ZK_P1), "n"(ZK_P2), "n"(ZK_P3), "n"(ZK_P4), "n"(ZK_P5), "n"(ZK_P6),
              "n"(ZK_P7));
        // shift down one limb; the carry and the next input limb (hi) form the new t[8]
        t[0] = t[1]; t[1] = t[2]; t[2] = t[3]; t[3] = t[4]; t[4] = t[5]; t[5] = t[6]; t[6] = t[7]; t[7] = t[8];
        t[8] = carry + (i == 0 ? hi : 0u);
    }
    fr_t r;
#pragma unroll
    for (int i = 0; i < 8; i++) r.v[i] = t[i];
    // T < 2^300 ⇒ result < 2^44 + p < 2p; t[8] == 0
    return fr_reduce_once(r);
}

// ---------------------------------------------------------------- conversions
__device__ __forceinline__ fr_t fr_from_u32(uint32_t x) {      // Montgomery form of a small integer
    fr_t b = fr_zero();
    b.v[0] = x;
    return fr_mul(ZK_R2, b);
}
__device__ __forceinline__ fr_t fr_from_i32(int32_t x) {
    fr_t a = fr_from_u32(x < 0 ? (uint32_t)(-(int64_t)x) : (uint32_t)x);
    return x < 0 ? fr_neg(a) : a;
}
__device__ __forceinline__ fr_t fr_to_canonical(const fr_t& a) {   // Montgomery -> integer in [0, p)
    fr_t one = fr_zero();
    one.v[0] = 1;
    return fr_mul(a, one);
}
__device__ __forceinline__ fr_t fr_to_canonical_cold(const fr_t& a) {
    fr_t one = fr_zero();
    one.v[0] = 1;
    return fr_mul_cold(a, one);
}
__device__ __forceinline__ fr_t fr_from_canonical(const fr_t& x) {  // integer < 2^256 -> Montgomery
    return fr_mul(ZK_R2, x);
}
// a * small unsigned integer k (k < 2^32)
__device__ __forceinline__ fr_t fr_mul_u32(const fr_t& a, uint32_t k) {
    fr_t b = fr_zero();
    b.v[0] = k;
    return fr_mul(fr_mul(a, ZK_R2), b);
}

// ---------------------------------------------------------------- memory access
__device__ __forceinline__ fr_t fr_load(const fr_t* p) {
    const uint4* q = reinterpret_cast<const uint4*>(p);
    uint4 x = __ldg(q), y = __ldg(q + 1);
    return fr_t{{x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w}};
}
__device__ __forceinline__ fr_t fr_load_cg(const fr_t* p) {   // streaming (not kept in L1)
    const uint4* q = reinterpret_cast<const uint4*>(p);
    uint4 x = __ldcs(q), y = __ldcs(q + 1);
    return fr_t{{x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w}};
}
__device__ __forceinline__ fr_t fr_load_l2(const fr_t* p) {   // bypass L1: data written earlier in the same kernel
    const uint4* q = reinterpret_cast<const uint4*>(p);
    uint4 x = __ldcg(q), y = __ldcg(q + 1);
    return fr_t{{x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w}};
}
__device__ __forceinline__ void fr_store(fr_t* p, const fr_t& a) {
    uint4* q = reinterpret_cast<uint4*>(p);
    q[0] = make_uint4(a.v[0], a.v[1], a.v[2], a.v[3]);
    q[1] = make_uint4(a.v[4], a.v[5], a.v[6], a.v[7]);
}
__device__ __forceinline__ fr_t fr_shfl_down(const fr_t& a, int delta) {
    fr_t r;
#pragma unroll
    for (int i = 0; i < 8; i++) r.v[i] = __shfl_down_sync(0xffffffffu, a.v[i], delta);
    return r;
}
__device__ __forceinline__ fr_t fr_shfl_xor(const fr_t& a, int mask, unsigned lanes = 0xffffffffu) {
    fr_t r;
#pragma unroll
    for (int i = 0; i < 8; i++) r.v[i] = __shfl_xor_sync(lanes, a.v[i], mask);
    return r;
}
// m * e for a small integer m in [-3, 3] (selects and additions, no multiplication, no branches)
__device__ __forceinline__ fr_t fr_mul_small(const fr_t& e, int m) {
    const int am = m < 0 ? -m : m;
    const fr_t e2 = fr_add(e, e);
    fr_t r = fr_zero(), t = fr_zero();
#pragma unroll
    for (int i = 0; i < 8; i++) {
        r.v[i] = (am & 1) ? e.v[i] : 0u;
        t.v[i] = (am & 2) ? e2.v[i] : 0u;
    }
    r = fr_add(r, t);
    const fr_t n = fr_neg(r);
#pragma unroll
    for (int i = 0; i < 8; i++) r.v[i] = m < 0 ? n.v[i] : r.v[i];
    return r;
}

// Fermat inverse a^(p-2) (single thread; used only for a handful of scalars)
// a^-1 (Montgomery in, Montgomery out) by the binary extended Euclidean algorithm on the stored integer
// A = aR (< p): x = A^-1 mod p, then mont(x, R^3) = A^-1 R^2 = a^-1 R.  ~700 shift / subtract steps on 4 x 64-bit
// limbs instead of ~380 products of the Fermat chain (variable time: for public values only).  a != 0.
__device__ inline void u4_shr1(uint64_t (&x)[4]) {
    x[0] = (x[0] >> 1) | (x[1] << 63);
    x[1] = (x[1] >> 1) | (x[2] << 63);
    x[2] = (x[2] >> 1) | (x[3] << 63);
    x[3] >>= 1;
}
__device__ inline void u4_add(uint64_t (&x)[4], const uint64_t (&y)[4]) {   // x += y (no overflow past 2^256)
    uint64_t c = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const uint64_t s = x[i] + y[i];
        const uint64_t c1 = s < x[i];
        x[i] = s + c;
        c = c1 | (x[i] < s);
    }
}
__device__ inline bool u4_sub(uint64_t (&x)[4], const uint64_t (&y)[4]) {   // x -= y, returns the borrow
    uint64_t b = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const uint64_t d = x[i] - y[i];
        const uint64_t b1 = x[i] < y[i];
        x[i] = d - b;
        b = b1 | (d < b);
    }
    return b != 0;
}
__device__ inline bool u4_ge(const uint64_t (&x)[4], const uint64_t (&y)[4]) {
    for (int i = 3; i >= 0; i--)
        if (x[i] != y[i]) return x[i] > y[i];
    return true;
}
__device__ inline bool u4_is_one(const uint64_t (&x)[4]) { return x[0] == 1 && !x[1] && !x[2] && !x[3]; }
__device__ inline fr_t fr_inv_bgcd(const fr_t& a) {
    const uint64_t P[4] = {((uint64_t)ZK_P1 << 32) | ZK_P0, ((uint64_t)ZK_P3 << 32) | ZK_P2, ((uint64_t)ZK_P5 << 32) | ZK_P4,
                           ((uint64_t)ZK_P7 << 32) | ZK_P6};
    uint64_t u[4], v[4] = {P[0], P[1], P[2], P[3]}, x1[4] = {1, 0, 0, 0}, x2[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 4; i++) u[i] = ((uint64_t)a.v[2 * i + 1] << 32) | a.v[2 * i];
    // invariant: x1 A = u, x2 A = v (mod p); x1, x2 < p
    while (!u4_is_one(u) && !u4_is_one(v)) {
        while (!(u[0] & 1)) {
            u4_shr1(u);
            if (x1[0] & 1) u4_add(x1, P);   // x1 + p < 2^256 (p < 2^255)
            u4_shr1(x1);
        }
        while (!(v[0] & 1)) {
            u4_shr1(v);
            if (x2[0] & 1) u4_add(x2, P);
            u4_shr1(x2);
        }
        if (u4_ge(u, v)) {
            u4_sub(u, v);
            if (u4_sub(x1, x2)) u4_add(x1, P);
        } else {
            u4_sub(v, u);
            if (u4_sub(x2, x1)) u4_add(x2, P);
        }
    }
    const uint64_t* x = u4_is_one(u) ? x1 : x2;
    fr_t r;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        r.v[2 * i] = (uint32_t)x[i];
        r.v[2 * i + 1] = (uint32_t)(x[i] >> 32);
    }
    return fr_mul(r, ZK_R3);
}

__device__ inline fr_t fr_inv(const fr_t& a) {
    // p - 2: the low limb 0x00000001 borrows from the next one
    const uint32_t e[8] = {0xffffffffu, ZK_P1 - 1, ZK_P2, ZK_P3, ZK_P4, ZK_P5, ZK_P6, ZK_P7};
    fr_t r = fr_one();
    for (int i = 7; i >= 0; i--)
        for (int b = 31; b >= 0; b--) {
            r = fr_sqr(r);
            if ((e[i] >> b) & 1) r = fr_mul(r, a);
        }
    return r;
}

}  // namespace zk
