// sumcheck.cu — aggregated product sumcheck (Protocol 3 P:L504-527).
//
// Statement: claim = sum_{x in {0,1}^m} beta(w, x_{<n_eq}) prod_{k<K} T_k(x), variables bound LSB first (D2).
// Round t, pair b = (T[2b], T[2b+1]) of the current tables; message = evaluations at X = 0..K of
//   f_t(X) = sum_b beta(w_{t+1..n_eq-1}, b) prod_k (T_k[2b] + X (T_k[2b+1] - T_k[2b]))     (t < n_eq, D4)
//   g_t(X) = sum_b prod_k (...)                                                            (t >= n_eq)
// One kernel per round fuses: the fold of every table by r_{t-1} (row a5: reads 4 elements per pair,
// writes the 2 folded ones to a ping-pong buffer), the suffix-eq weight of the pair, the K+1
// evaluations, a warp-shuffle + block-tree + last-block grid reduction, and the Fiat-Shamir step on
// the device (absorb the message, squeeze r_t) — no host synchronisation inside a sumcheck.
//
// Suffix eq weights without materialising 2^n_eq entries: E_t(b) = LO_t[b mod 2^l] * HI[(b >> l) mod 2^h]
// with HI = beta(w_{n_eq-h..n_eq-1}, .) (h <= 10) fixed and LO_t = beta(w_{t+1..n_eq-h-1}, .).  Because
// beta(w_s, 0) + beta(w_s, 1) = 1, LO_{t+1}[c] = LO_t[2c] + LO_t[2c+1]: the round kernel writes the next
// LO level with additions only.  Once LO is exhausted the HI table is pair-summed the same way.
#include <cstdlib>
#include <cstdio>
#include <vector>

#include "sumcheck.cuh"
#include "tables.cuh"

namespace zk {

struct ScRoundArgs {
    const fr_t* src[3];
    fr_t* dst[3];
    uint64_t n_pairs;
    const fr_t* r_prev;      // r_{t-1} (Montgomery) when folding
    // eq weights: mode 0 none, 1 split (cur = LO level, hi = HI), 2 single table (cur)
    int eq_mode;
    const fr_t* eq_cur;
    const fr_t* eq_hi;
    fr_t* eq_next;
    uint32_t lo_cnt;         // number of variables in the current LO (mode 1) or current table (mode 2)
    uint32_t hb;             // variables in HI (mode 1)
    // reduction + finalize
    fr_t* partials;
    unsigned int* ticket;
    uint8_t* st;
    uint32_t t, n_eq;
    const fr_t* w;           // device w (Montgomery), for the claim of round 0
    fr_t* claim;             // device claim (Montgomery)
    int compute_claim;       // round 0 only: derive the claim from the message and absorb it
    uint8_t* claim_bytes;    // canonical claim in the proof
    uint8_t* msg_out;        // canonical message bytes in the proof
    fr_t* r_out;             // r_t (Montgomery)
    uint8_t* point_out;      // r_t canonical
    fr_t* part_out;          // sharded mode: write the (scaled) K+1 totals here instead of the transcript step
    const fr_t* scale;       // sharded mode: the rank's eq factor over its high bits (nullptr = 1)
    // running claim (single-device provers): c_t in, c_{t+1} = f_t(r_t) out after the challenge; the derived-X=1
    // rounds (k_sc_round2f MODE bit 2) take f_t(1) from it: (c_t - (1 - w_t) f_t(0)) w_t^-1, or c_t - f_t(0)
    fr_t* run_claim;
    const fr_t* winv;        // w_t^-1 for every t < n_eq (derived rounds under the eq factor)
};

// Finalizer of a product-sumcheck round (last block, warp 0): the claim of round 0 (when computed),
// the message, the transcript step; in sharded mode the rank's (scaled) totals instead.
__device__ __noinline__ void sc_finish(const ScRoundArgs& a, const fr_t* tot, const int K) {
    __shared__ FsScratch fs;
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    if (a.part_out) {
        if (lane <= K) {
            fr_t v = tot[lane & 3];
            if (a.scale) v = fr_mul_cold(v, fr_load(a.scale));
            fr_store(&a.part_out[lane], v);
        }
        return;
    }
    fs_begin(fs, a.st);
    if (a.compute_claim) {
        __shared__ fr_t claim_sm;
        if (lane == 0) {
            fr_t c;
            if (a.t < a.n_eq) {
                fr_t w0 = fr_load(&a.w[a.t]);
                c = fr_add(fr_mul_cold(fr_sub(fr_one(), w0), tot[0]), fr_mul_cold(w0, tot[1]));
            } else {
                c = fr_add(tot[0], tot[1]);
            }
            fr_store(a.claim, c);
            claim_sm = c;
        }
        __syncwarp();
        fs_absorb_frs(fs, "sc/claim", claim_sm, 1, a.claim_bytes);
    }
    fs_absorb_frs(fs, "sc/msg", lane <= K ? tot[lane & 3] : fr_zero(), K + 1, a.msg_out);
    fr_t rt = fs_challenge(fs, "sc/r");
    if (lane == 0) {
        fr_store(a.r_out, rt);
        fr_canon_to_bytes(fs.rc, a.point_out);
        if (a.run_claim) {   // c_{t+1} = f_t(r_t) (Lagrange through the message's K + 1 points)
            fr_t e[4];
            for (int x = 0; x <= K; x++) e[x] = tot[x];
            fr_store(a.run_claim, interp_small(e, K, rt));
        }
    }
    fs_end(fs, a.st);
}

template <int K, bool FOLD>
__global__ void __launch_bounds__(256) k_sc_round(ScRoundArgs a) {
    fr_t acc[K + 1];
#pragma unroll
    for (int x = 0; x <= K; x++) acc[x] = fr_zero();
    fr_t r;
    if (FOLD) r = fr_load(a.r_prev);
    const uint64_t lo_mask = (1ull << a.lo_cnt) - 1, hi_mask = (1ull << a.hb) - 1;
    const uint64_t next_count = a.lo_cnt ? (1ull << (a.lo_cnt - 1)) : 0;
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < a.n_pairs;
         b += (uint64_t)gridDim.x * blockDim.x) {
        fr_t lo[K], d[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            fr_t v0, v1;
            if (FOLD) {
                const fr_t* s = a.src[k] + 4 * b;
                fr_t x0 = fr_load_cg(s), x1 = fr_load_cg(s + 1), x2 = fr_load_cg(s + 2), x3 = fr_load_cg(s + 3);
                v0 = fr_add(x0, fr_mul(r, fr_sub(x1, x0)));
                v1 = fr_add(x2, fr_mul(r, fr_sub(x3, x2)));
                fr_store(a.dst[k] + 2 * b, v0);
                fr_store(a.dst[k] + 2 * b + 1, v1);
            } else {
                v0 = fr_load_cg(a.src[k] + 2 * b);
                v1 = fr_load_cg(a.src[k] + 2 * b + 1);
            }
            lo[k] = v0;
            d[k] = fr_sub(v1, v0);
        }
        // suffix eq weight of this pair
        fr_t e;
        bool has_e = a.eq_mode != 0;
        if (a.eq_mode == 1) {
            e = fr_mul(fr_load(&a.eq_cur[b & lo_mask]), fr_load(&a.eq_hi[(b >> a.lo_cnt) & hi_mask]));
        } else if (a.eq_mode == 2) {
            e = fr_load(&a.eq_cur[b & lo_mask]);
        }
        if (a.eq_mode && b < next_count)
            fr_store(&a.eq_next[b], fr_add(fr_load(&a.eq_cur[2 * b]), fr_load(&a.eq_cur[2 * b + 1])));
        // evaluations at X = 0..K: v_k(X) = lo_k + X d_k
        fr_t v[K];
#pragma unroll
        for (int k = 0; k < K; k++) v[k] = lo[k];
#pragma unroll
        for (int x = 0; x <= K; x++) {
            fr_t p = v[0];
#pragma unroll
            for (int k = 1; k < K; k++) p = fr_mul(p, v[k]);
            if (has_e) p = fr_mul(p, e);
            acc[x] = fr_add(acc[x], p);
            if (x < K)
#pragma unroll
                for (int k = 0; k < K; k++) v[k] = fr_add(v[k], d[k]);
        }
    }
    __shared__ fr_t tot[K + 1];
    if (grid_reduce_fr_block<K + 1>(acc, a.partials, a.ticket, tot)) sc_finish(a, tot, K);
}

// Factored K = 2 round (the large statements: C5, the sharded prover).  Pairs are grouped by their
// HI index (b >> lo_cnt): inside a group the suffix eq weight is E'(b) = LO[b mod 2^lo_cnt] * HI[group],
// so a CTA accumulates LO-weighted sums over a slice of one group and multiplies its three totals by
// HI[group] once (no per-pair eq product).  Per pair: y = E' A at X = 0, 1 (two products), then
// P(0) = y0 B0, P(1) = y1 B1, P(inf) = (y1 - y0)(B1 - B0) (three products); the message evaluations are
// f(0) = P(0), f(1) = P(1), f(2) = 2 P(1) + 2 P(inf) - P(0).  With the fold (4 products) that is 9 Fr
// products per pair against 11 (no eq: 4 + 3 against 4 + 3).  MODE 0: round 0 from Fr tables; 1: fold
// rounds; 2: round 0 from int32 tables, embedded on the fly (a product with a one-limb operand, half a
// full product) and written out for round 1 — no separate embedding pass.
struct fr4_t { fr_t a, b, c, d; };
// four int32 -> Montgomery embeddings (each a product with a one-limb operand: half a full product)
static __device__ __noinline__ fr4_t fr_embed4_ni(int32_t x, int32_t y, int32_t z, int32_t w) {
    return fr4_t{fr_from_i32(x), fr_from_i32(y), fr_from_i32(z), fr_from_i32(w)};
}

struct Sc2Args {
    ScRoundArgs r;            // tables, eq (LO = eq_cur, HI = eq_hi or null), reduction, finalize
    const int32_t* i32[2];    // MODE 2 sources
    fr_t* emb[2];             // MODE 2: embedded tables written here
    uint32_t slices;          // CTAs per group when there are fewer groups than CTAs
    int flat;                 // groups too small for a CTA: every pair applies its HI value itself
};

// ---- integer round 0 for int32 tables (C5, the sharded prover): the pair products are exact integers
// P(0) = a0 b0, P(1) = a1 b1, P(inf) = (a1 - a0)(b1 - b0) (|P| < 2^64), so round 0 needs no field product
// per pair: E' P is accumulated lazily as a 352-bit integer (u = P + 2^64 in [0, 2^65): 16 IMAD.WIDE),
// the bias 2^64 sum E' is removed once per work item, and one Montgomery reduction closes each sum.
__device__ __forceinline__ void mac65(uint32_t (&acc)[11], const fr_t& e, unsigned __int128 u) {
    const uint32_t lo = (uint32_t)u, hi = (uint32_t)(u >> 32), top = (uint32_t)(u >> 64);
    uint64_t C = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const uint64_t t = (uint64_t)e.v[j] * lo + acc[j] + C;
        acc[j] = (uint32_t)t;
        C = t >> 32;
    }
#pragma unroll
    for (int j = 8; j < 11; j++) {
        const uint64_t t = (uint64_t)acc[j] + C;
        acc[j] = (uint32_t)t;
        C = t >> 32;
    }
    C = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const uint64_t t = (uint64_t)e.v[j] * hi + acc[j + 1] + C;
        acc[j + 1] = (uint32_t)t;
        C = t >> 32;
    }
#pragma unroll
    for (int j = 9; j < 11; j++) {
        const uint64_t t = (uint64_t)acc[j] + C;
        acc[j] = (uint32_t)t;
        C = t >> 32;
    }
    if (top) {
        C = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint64_t t = (uint64_t)e.v[j] + acc[j + 2] + C;
            acc[j + 2] = (uint32_t)t;
            C = t >> 32;
        }
        acc[10] += (uint32_t)C;
    }
}
__device__ __forceinline__ void add9(uint32_t (&s)[9], const fr_t& e) {
    uint64_t C = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const uint64_t t = (uint64_t)s[j] + e.v[j] + C;
        s[j] = (uint32_t)t;
        C = t >> 32;
    }
    s[8] += (uint32_t)C;
}
// Montgomery reduction of an 11-limb integer T (< p 2^256): T R^{-1} mod p.  T = lo9 + w9 2^288 + w10 2^320 and
// 2^288 R^{-1} = 2^32, 2^320 R^{-1} = 2^64, so REDC(T) = REDC(lo9) + (w9 2^32 + w10 2^64) (the second term
// < 2^96 < p; fr_redc_wide's top limb stays zero, so its carry into t[8] cannot wrap)
__device__ __noinline__ fr_t fr_redc11(const uint32_t (&w)[11]) {
    const uint32_t lo[10] = {w[0], w[1], w[2], w[3], w[4], w[5], w[6], w[7], w[8], 0};
    const fr_t x = fr_redc_wide(lo);
    return fr_add(x, fr_t{{0, w[9], w[10], 0, 0, 0, 0, 0}});
}

// Round 1 after the integer round 0: the fold v0 + r (v1 - v0) of an int32 pair, straight to Montgomery
// form.  With u = v + 2^31 in [0, 2^32):  x = (1 - r) u0 + r u1 - 2^31, so
//     I = u0 [(1 - r) R^2] + u1 [r R^2] + [-2^31 R^2]     (residues < p; I < 2^33 p < 2^300)
// and REDC(I) = x R: two 32 x 256-bit multiply-accumulates and one reduction per value instead of two
// half products.  Out of line, two values per call (a small body shared by both call sites: I-cache).
struct FoldI32 { fr_t omr2, r2, cneg; };
__device__ __forceinline__ void mac32(uint32_t (&w)[10], const fr_t& e, uint32_t u) {
    uint64_t C = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const uint64_t t = (uint64_t)e.v[j] * u + w[j] + C;
        w[j] = (uint32_t)t;
        C = t >> 32;
    }
    const uint64_t t = (uint64_t)w[8] + C;
    w[8] = (uint32_t)t;
    w[9] += (uint32_t)(t >> 32);
}
__device__ __forceinline__ fr_t fold_i32(const FoldI32& f, int32_t v0, int32_t v1) {
    uint32_t w[10] = {f.cneg.v[0], f.cneg.v[1], f.cneg.v[2], f.cneg.v[3], f.cneg.v[4], f.cneg.v[5], f.cneg.v[6],
                      f.cneg.v[7], 0, 0};
    mac32(w, f.omr2, (uint32_t)v0 ^ 0x80000000u);
    mac32(w, f.r2, (uint32_t)v1 ^ 0x80000000u);
    return fr_redc_wide(w);
}
struct fr2_t { fr_t a, b; };
static __device__ __noinline__ fr2_t fold2_i32_ni(const FoldI32& f, int4 x) {   // two values per call: a small body
    return fr2_t{fold_i32(f, x.x, x.y), fold_i32(f, x.z, x.w)};
}

// Montgomery form of 2^64 (= 2^64 R mod p), derived with Python integers
#define ZK_MONT_2_64 fr_const(0x0121c884u, 0xc98da28eu, 0xc7363c67u, 0xe6f4f4a0u, 0xe92e7df1u, 0xb2d6ebc4u, 0x9d26242au, 0x19ae5794u)

// Round 0 from int32 tables, grouped eq weights (E' = LO[j], HI[group] once per item): the sums of E' P(0),
// E' P(1), E' P(inf) as exact lazy integers.  Writes nothing but the next LO level; round 1 folds from the
// int32 tables (MODE 3 of k_sc_round2f).
__global__ void __launch_bounds__(256, 2) k_sc_round0_int(Sc2Args A) {
    const ScRoundArgs& a = A.r;
    const uint32_t lo_cnt = a.lo_cnt;
    const uint64_t ngroups = a.n_pairs >> lo_cnt ? a.n_pairs >> lo_cnt : 1;
    const uint64_t gsize = a.n_pairs < (1ull << lo_cnt) ? a.n_pairs : (1ull << lo_cnt);
    const uint64_t slices = A.slices;
    const uint64_t slice_len = (gsize + slices - 1) / slices;
    const uint64_t next_count = lo_cnt ? (1ull << (lo_cnt - 1)) : 0;
    const uint64_t hi_mask = (1ull << a.hb) - 1, lo_mask = (1ull << lo_cnt) - 1;
    const int2* ia = reinterpret_cast<const int2*>(A.i32[0]);
    const int2* ib = reinterpret_cast<const int2*>(A.i32[1]);
    fr_t tot[3] = {fr_zero(), fr_zero(), fr_zero()};
    for (uint64_t item = blockIdx.x; item < ngroups * slices; item += gridDim.x) {
        const uint64_t g = item / slices, sl = item % slices;
        const uint64_t j_end = (sl + 1) * slice_len < gsize ? (sl + 1) * slice_len : gsize;
        uint32_t acc[3][11], S[9];
#pragma unroll
        for (int v = 0; v < 3; v++)
#pragma unroll
            for (int i = 0; i < 11; i++) acc[v][i] = 0;
#pragma unroll
        for (int i = 0; i < 9; i++) S[i] = 0;
        bool any = false;
        for (uint64_t j = sl * slice_len + threadIdx.x; j < j_end; j += blockDim.x) {
            any = true;
            const uint64_t b = (g << lo_cnt) + j;
            const int2 x = __ldcs(ia + b), y = __ldcs(ib + b);
            const fr_t e = fr_load(&a.eq_cur[b & lo_mask]);
            if (b < next_count)
                fr_store(&a.eq_next[b], fr_add(fr_load(&a.eq_cur[2 * b]), fr_load(&a.eq_cur[2 * b + 1])));
            const unsigned __int128 bias = (unsigned __int128)1 << 64;
            const __int128 p0 = (__int128)((int64_t)x.x * y.x), p1 = (__int128)((int64_t)x.y * y.y);
            const __int128 pi = (__int128)((int64_t)x.y - x.x) * (__int128)((int64_t)y.y - y.x);
            mac65(acc[0], e, (unsigned __int128)p0 + bias);
            mac65(acc[1], e, (unsigned __int128)p1 + bias);
            mac65(acc[2], e, (unsigned __int128)pi + bias);
            add9(S, e);
        }
        if (any) {   // sum E' P = REDC(acc) - 2^64 REDC(S), to Montgomery form (x R^2), times HI[group]
            const uint32_t s10[10] = {S[0], S[1], S[2], S[3], S[4], S[5], S[6], S[7], S[8], 0};
            const fr_t sb = fr_mul(fr_redc_wide(s10), ZK_MONT_2_64);   // 2^64 sum E' (plain)
            const fr_t h = a.eq_hi ? fr_mul(fr_load(&a.eq_hi[g & hi_mask]), ZK_R2) : ZK_R2;   // HI R (or R)
#pragma unroll
            for (int v = 0; v < 3; v++) tot[v] = fr_add(tot[v], fr_mul(fr_sub(fr_redc11(acc[v]), sb), h));
        }
    }
    __shared__ fr_t tt[3];
    __shared__ fr_t msg[3];
    if (grid_reduce_fr_block<3>(tot, a.partials, a.ticket, tt)) {
        if (threadIdx.x == 0) {   // evaluations at X = 0, 1, 2 of the quadratic with P(0), P(1), P(inf)
            msg[0] = tt[0];
            msg[1] = tt[1];
            msg[2] = fr_sub(fr_dbl(fr_add(tt[1], tt[2])), tt[0]);
        }
        __syncthreads();
        sc_finish(a, msg, 2);
    }
}
// the factored K = 2 rounds' product groups (ZKDL_SC_MULW): 3 = the two- and three-product bodies
// (interleaved chains), 1 = single-product body calls (the smaller body stays in the L0 instruction cache:
// C5 m = 26 10.1 -> 9.0 ms, m = 24 3.64 -> 3.34 ms, same proofs)
#ifndef ZKDL_SC_MULW
#define ZKDL_SC_MULW 1
#endif
__device__ __forceinline__ fr3_t sc_mul3(const fr_t& a0, const fr_t& b0, const fr_t& a1, const fr_t& b1, const fr_t& a2,
                                         const fr_t& b2) {
#if ZKDL_SC_MULW == 3
    return fr_mul3_ni(a0, b0, a1, b1, a2, b2);
#elif ZKDL_SC_MULW == 2
    const fr2p_t p = fr_mul2_ni(a0, b0, a1, b1);
    return fr3_t{p.x, p.y, fr_mul_ni(a2, b2)};
#else
    return fr3_t{fr_mul_ni(a0, b0), fr_mul_ni(a1, b1), fr_mul_ni(a2, b2)};
#endif
}
__device__ __forceinline__ fr2p_t sc_mul2(const fr_t& a0, const fr_t& b0, const fr_t& a1, const fr_t& b1) {
#if ZKDL_SC_MULW >= 2
    return fr_mul2_ni(a0, b0, a1, b1);
#else
    return fr2p_t{fr_mul_ni(a0, b0), fr_mul_ni(a1, b1)};
#endif
}

template <int MODE>
__global__ void __launch_bounds__(256, 2) k_sc_round2f(Sc2Args A) {
    const ScRoundArgs& a = A.r;
    constexpr bool FOLD = (MODE & 3) == 1 || (MODE & 3) == 3;   // MODE 3: round 1 folding straight from the int32 tables
    constexpr bool DER = MODE & 4;   // f(1) derived in the finalizer from the running claim: P(0), P(inf) only
    const bool has_e = a.eq_mode != 0;
    const uint32_t lo_cnt = has_e ? a.lo_cnt : 0;
    // pairs per group (log2): the LO range; without eq weights the whole round is one group
    const uint32_t gsize_log = has_e ? lo_cnt : 63 - __clzll(a.n_pairs);
    const uint64_t ngroups = a.n_pairs >> gsize_log ? a.n_pairs >> gsize_log : 1;
    uint64_t gsize = a.n_pairs < (1ull << gsize_log) ? a.n_pairs : (1ull << gsize_log);
    if (A.flat) gsize = a.n_pairs;   // one group; E' = LO[b mod 2^lo_cnt] * HI[b >> lo_cnt] per pair
    const uint64_t slices = A.slices;
    const uint64_t slice_len = (gsize + slices - 1) / slices;
    const uint64_t next_count = lo_cnt ? (1ull << (lo_cnt - 1)) : 0;
    const uint64_t hi_mask = (1ull << a.hb) - 1;
    fr_t r;
    if (FOLD) r = fr_load(a.r_prev);
    FoldI32 fi;
    if ((MODE & 3) == 3) {   // residues (1 - r) R^2, r R^2, -2^31 R^2 (fr_mul(x R, R^2) = x R^2)
        fi.r2 = fr_mul(r, ZK_R2);
        fi.omr2 = fr_mul(fr_sub(fr_one(), r), ZK_R2);
        fi.cneg = fr_mul(fr_neg(fr_from_u32(0x80000000u)), ZK_R2);
    }
    fr_t tot0 = fr_zero(), tot1 = fr_zero(), toti = fr_zero();
    const uint64_t nitems = (A.flat ? 1 : ngroups) * slices;
    const uint64_t lo_mask = (1ull << lo_cnt) - 1;
    for (uint64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
        const uint64_t g = item / slices, sl = item % slices;
        const uint64_t j_end = (sl + 1) * slice_len < gsize ? (sl + 1) * slice_len : gsize;
        fr_t s0 = fr_zero(), s1 = fr_zero(), si = fr_zero();
        bool any = false;
        for (uint64_t j = sl * slice_len + threadIdx.x; j < j_end; j += blockDim.x) {
            any = true;
            const uint64_t b = A.flat ? j : (g << gsize_log) + j;
            // products in three-wide out-of-line groups (three independent CIOS chains per call, one
            // ~24 KB body shared by every call site: the inlined 9-product loop missed the I-cache)
            fr_t a0, a1, b0, b1, e;
            const fr_t zero = fr_zero();
            if (has_e) {
                e = fr_load(&a.eq_cur[b & lo_mask]);
                if (b < next_count)
                    fr_store(&a.eq_next[b], fr_add(fr_load(&a.eq_cur[2 * b]), fr_load(&a.eq_cur[2 * b + 1])));
            }
            fr3_t q;   // second group: (r db, E' a0, E' a1) in folding rounds with eq weights
            bool q_done = false;
            if (FOLD) {
                fr_t x0, x1, x2, x3, z0, z1, z2, z3;
                if constexpr ((MODE & 3) == 3) {   // fold straight from the int32 tables (fold4_i32_ni)
                    const int4 ia = __ldcs(reinterpret_cast<const int4*>(A.i32[0]) + b);
                    const int4 ib = __ldcs(reinterpret_cast<const int4*>(A.i32[1]) + b);
                    const fr2_t fa = fold2_i32_ni(fi, ia), fb = fold2_i32_ni(fi, ib);
                    a0 = fa.a;
                    a1 = fa.b;
                    b0 = fb.a;
                    b1 = fb.b;
                    (void)x0; (void)x1; (void)x2; (void)x3; (void)z0; (void)z1; (void)z2; (void)z3;
                } else {
                const fr_t* sa = a.src[0] + 4 * b;
                const fr_t* sb = a.src[1] + 4 * b;
                x0 = fr_load_cg(sa); x1 = fr_load_cg(sa + 1); x2 = fr_load_cg(sa + 2); x3 = fr_load_cg(sa + 3);
                z0 = fr_load_cg(sb); z1 = fr_load_cg(sb + 1); z2 = fr_load_cg(sb + 2); z3 = fr_load_cg(sb + 3);
                const fr3_t f = sc_mul3(r, fr_sub(x1, x0), r, fr_sub(x3, x2), r, fr_sub(z1, z0));
                a0 = fr_add(x0, f.x);
                a1 = fr_add(x2, f.y);
                b0 = fr_add(z0, f.z);
                if (has_e && !(A.flat && a.eq_hi)) {
                    q = sc_mul3(r, fr_sub(z3, z2), e, a0, e, DER ? fr_sub(a1, a0) : a1);
                    b1 = fr_add(z2, q.x);
                    q_done = true;
                } else {
                    const fr_t hh = (has_e && A.flat && a.eq_hi) ? fr_load(&a.eq_hi[(b >> lo_cnt) & hi_mask]) : zero;
                    const fr2p_t g2 = sc_mul2(r, fr_sub(z3, z2), e, hh);
                    b1 = fr_add(z2, g2.x);
                    if (has_e) e = g2.y;
                }
                }
                if constexpr ((MODE & 3) == 3) {
                    if (has_e && A.flat && a.eq_hi) e = fr_mul_ni(e, fr_load(&a.eq_hi[(b >> lo_cnt) & hi_mask]));
                }
                fr_store(a.dst[0] + 2 * b, a0);
                fr_store(a.dst[0] + 2 * b + 1, a1);
                fr_store(a.dst[1] + 2 * b, b0);
                fr_store(a.dst[1] + 2 * b + 1, b1);
            } else {
                if ((MODE & 3) == 2) {
                    const int2 ia = __ldcs(reinterpret_cast<const int2*>(A.i32[0]) + b);
                    const int2 ib = __ldcs(reinterpret_cast<const int2*>(A.i32[1]) + b);
                    const fr4_t em = fr_embed4_ni(ia.x, ia.y, ib.x, ib.y);
                    a0 = em.a;
                    a1 = em.b;
                    b0 = em.c;
                    b1 = em.d;
                    fr_store(A.emb[0] + 2 * b, a0);
                    fr_store(A.emb[0] + 2 * b + 1, a1);
                    fr_store(A.emb[1] + 2 * b, b0);
                    fr_store(A.emb[1] + 2 * b + 1, b1);
                } else {
                    a0 = fr_load_cg(a.src[0] + 2 * b);
                    a1 = fr_load_cg(a.src[0] + 2 * b + 1);
                    b0 = fr_load_cg(a.src[1] + 2 * b);
                    b1 = fr_load_cg(a.src[1] + 2 * b + 1);
                }
                if (has_e && A.flat && a.eq_hi) e = fr_mul_ni(e, fr_load(&a.eq_hi[(b >> lo_cnt) & hi_mask]));
            }
            if constexpr (DER) {   // y0 = E' a0, yd = E' (a1 - a0); P(0) = y0 b0, P(inf) = yd (b1 - b0)
                fr_t y0 = a0, yd = fr_sub(a1, a0);
                if (has_e) {
                    if (q_done) {
                        y0 = q.y;
                        yd = q.z;
                    } else {
                        const fr2p_t q2 = sc_mul2(e, a0, e, yd);
                        y0 = q2.x;
                        yd = q2.y;
                    }
                }
                const fr2p_t p = sc_mul2(y0, b0, yd, fr_sub(b1, b0));
                s0 = fr_add(s0, p.x);
                si = fr_add(si, p.y);
                continue;
            }
            fr_t y0 = a0, y1 = a1;
            if (has_e) {
                if (q_done) {
                    y0 = q.y;
                    y1 = q.z;
                } else {   // two products only: the two-product body (no wasted third slot)
                    const fr2p_t q2 = sc_mul2(e, a0, e, a1);
                    y0 = q2.x;
                    y1 = q2.y;
                }
            }
            const fr3_t p = sc_mul3(y0, b0, y1, b1, fr_sub(y1, y0), fr_sub(b1, b0));
            s0 = fr_add(s0, p.x);
            s1 = fr_add(s1, p.y);
            si = fr_add(si, p.z);
        }
        if (any && has_e && a.eq_hi && !A.flat) {   // this group's HI factor, once per CTA and group
            const fr_t h = fr_load(&a.eq_hi[g & hi_mask]);
            s0 = fr_mul_ni(s0, h);
            s1 = fr_mul_ni(s1, h);
            si = fr_mul_ni(si, h);
        }
        tot0 = fr_add(tot0, s0);
        tot1 = fr_add(tot1, s1);
        toti = fr_add(toti, si);
    }
    fr_t acc[3] = {tot0, tot1, toti};
    __shared__ fr_t tt[3];
    __shared__ fr_t msg[3];
    if (grid_reduce_fr_block<3>(acc, a.partials, a.ticket, tt)) {
        if (threadIdx.x == 0) {   // evaluations at X = 0, 1, 2 of the quadratic with P(0), P(1), P(inf)
            msg[0] = tt[0];
            if (DER) {   // (1 - w_t) f(0) + w_t f(1) = c_t under the eq factor, f(0) + f(1) = c_t after it
                const fr_t c = fr_load_l2(a.run_claim);
                if (a.t < a.n_eq) {
                    const fr_t w = fr_load(&a.w[a.t]);
                    msg[1] = fr_mul_cold(fr_sub(c, fr_mul_cold(fr_sub(fr_one(), w), tt[0])), fr_load(&a.winv[a.t]));
                } else {
                    msg[1] = fr_sub(c, tt[0]);
                }
            } else {
                msg[1] = tt[1];
            }
            msg[2] = fr_sub(fr_dbl(fr_add(msg[1], tt[2])), tt[0]);
        }
        __syncthreads();
        sc_finish(a, msg, 2);
    }
}

// N2 (D22): Protocol 2's zero form for the aggregated Hadamard product.  Tables (Y, A, B); per pair the
// term p(X) = Y(X) - A(X) B(X) times the suffix eq weight (f_t form, D4) at X = 0, 1, 2; the claim is 0.
template <bool FOLD>
__global__ void __launch_bounds__(256) k_sc_zero_round(ScRoundArgs a) {
    fr_t acc[3] = {fr_zero(), fr_zero(), fr_zero()};
    fr_t r;
    if (FOLD) r = fr_load(a.r_prev);
    const uint64_t lo_mask = (1ull << a.lo_cnt) - 1, hi_mask = (1ull << a.hb) - 1;
    const uint64_t next_count = a.lo_cnt ? (1ull << (a.lo_cnt - 1)) : 0;
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < a.n_pairs; b += (uint64_t)gridDim.x * blockDim.x) {
        fr_t lo[3], d[3];
#pragma unroll
        for (int k = 0; k < 3; k++) {
            fr_t v0, v1;
            if (FOLD) {
                const fr_t* s = a.src[k] + 4 * b;
                const fr_t x0 = fr_load_cg(s), x1 = fr_load_cg(s + 1), x2 = fr_load_cg(s + 2), x3 = fr_load_cg(s + 3);
                v0 = fr_add(x0, fr_mul_ni(r, fr_sub(x1, x0)));
                v1 = fr_add(x2, fr_mul_ni(r, fr_sub(x3, x2)));
                fr_store(a.dst[k] + 2 * b, v0);
                fr_store(a.dst[k] + 2 * b + 1, v1);
            } else {
                v0 = fr_load_cg(a.src[k] + 2 * b);
                v1 = fr_load_cg(a.src[k] + 2 * b + 1);
            }
            lo[k] = v0;
            d[k] = fr_sub(v1, v0);
        }
        fr_t e = fr_one();
        const bool has_e = a.eq_mode != 0;
        if (a.eq_mode == 1) e = fr_mul_ni(fr_load(&a.eq_cur[b & lo_mask]), fr_load(&a.eq_hi[(b >> a.lo_cnt) & hi_mask]));
        else if (a.eq_mode == 2) e = fr_load(&a.eq_cur[b & lo_mask]);
        if (a.eq_mode && b < next_count)
            fr_store(&a.eq_next[b], fr_add(fr_load(&a.eq_cur[2 * b]), fr_load(&a.eq_cur[2 * b + 1])));
#pragma unroll
        for (int x = 0; x < 3; x++) {
            fr_t p = fr_sub(lo[0], fr_mul_ni(lo[1], lo[2]));
            if (has_e) p = fr_mul_ni(p, e);
            acc[x] = fr_add(acc[x], p);
            if (x < 2)
#pragma unroll
                for (int k = 0; k < 3; k++) lo[k] = fr_add(lo[k], d[k]);
        }
    }
    __shared__ fr_t tot[3];
    if (grid_reduce_fr_block<3>(acc, a.partials, a.ticket, tot)) sc_finish(a, tot, 2);
}

// header (+ provided claim) before round 0; one warp
__global__ void k_sc_header(uint8_t* st, Bytes256 hdr, const fr_t* claim, int absorb_claim, uint8_t* claim_bytes) {
    __shared__ FsScratch fs;
    // the 12 proof-header bytes precede the claim in the proof buffer (no pageable host copy)
    if (threadIdx.x < 12) claim_bytes[(int)threadIdx.x - 12] = hdr.b[threadIdx.x];
    fs_begin(fs, st);
    fs_absorb_bytes(fs, "sc/hdr", hdr.b, hdr.len);
    if (absorb_claim) fs_absorb_frs(fs, "sc/claim", fr_load(claim), 1, claim_bytes);
    fs_end(fs, st);
}

// finals T_k~(r) = T_k[0] + r_{m-1} (T_k[1] - T_k[0]) on the last 2-element tables; one warp
__global__ void k_sc_finals(const fr_t* t0, const fr_t* t1, const fr_t* t2, int K, const fr_t* r_last, uint8_t* st,
                            uint8_t* finals_bytes, fr_t* finals_mont) {
    __shared__ FsScratch fs;
    const int lane = threadIdx.x & 31;
    const fr_t* T = lane == 0 ? t0 : (lane == 1 ? t1 : t2);
    fr_t f = fr_zero();
    if (lane < K) {
        fr_t r = fr_load(r_last);
        fr_t a = fr_load(T), b = fr_load(T + 1);
        f = fr_add(a, fr_mul(r, fr_sub(b, a)));
        if (finals_mont) fr_store(&finals_mont[lane], f);
    }
    fs_begin(fs, st);
    fs_absorb_frs(fs, "sc/final", f, K, finals_bytes);
    fs_end(fs, st);
}


// Sum the G rank partials (rank order) and run the transcript step of round t (sharded mode, §8(e));
// one warp.  all: G x (K+1) Montgomery elements.
__global__ void k_sc_combine(const fr_t* all, uint32_t G, int K, uint32_t t, uint32_t n_eq, const fr_t* w, fr_t* claim,
                             int compute_claim, uint8_t* st, uint8_t* claim_bytes, uint8_t* msg_out, fr_t* r_out,
                             uint8_t* point_out) {
    __shared__ FsScratch fs;
    __shared__ fr_t tot[4];
    const int lane = threadIdx.x & 31;
    if (lane <= K) {
        fr_t v = fr_zero();
        for (uint32_t g = 0; g < G; g++) v = fr_add(v, fr_load(&all[(size_t)g * (K + 1) + lane]));
        tot[lane] = v;
    }
    __syncwarp();
    fs_begin(fs, st);
    if (compute_claim) {
        __shared__ fr_t claim_sm;
        if (lane == 0) {
            fr_t c;
            if (t < n_eq) {
                fr_t w0 = fr_load(&w[t]);
                c = fr_add(fr_mul_cold(fr_sub(fr_one(), w0), tot[0]), fr_mul_cold(w0, tot[1]));
            } else {
                c = fr_add(tot[0], tot[1]);
            }
            fr_store(claim, c);
            claim_sm = c;
        }
        __syncwarp();
        fs_absorb_frs(fs, "sc/claim", claim_sm, 1, claim_bytes);
    }
    fs_absorb_frs(fs, "sc/msg", lane <= K ? tot[lane & 3] : fr_zero(), K + 1, msg_out);
    fr_t rt = fs_challenge(fs, "sc/r");
    if (lane == 0) {
        fr_store(r_out, rt);
        fr_canon_to_bytes(fs.rc, point_out);
    }
    fs_end(fs, st);
}

template <int K>
static void launch_round(zk_ctx* ctx, bool fold, unsigned int grid, const ScRoundArgs& a) {
    if (fold)
        ZK_LAUNCH(ctx, (k_sc_round<K, true>), grid, 256, 0, a);
    else
        ZK_LAUNCH(ctx, (k_sc_round<K, false>), grid, 256, 0, a);
}

// ---------------------------------------------------------------- engine
void ScEngine::setup(const fr_t* const tables[3], uint32_t L_, uint32_t t0_, uint32_t n_eq_loc_) {
    factored = !(getenv("ZKDL_SC_V") && atoi(getenv("ZKDL_SC_V")) == 0);
    for (int k = 0; k < 3; k++) i32[k] = nullptr;   // set_i32 after setup (a continuation has none)
    int0_used = false;
    L = L_;
    t0 = t0_;
    t = t0_;
    n_eq_loc = n_eq_loc_;
    const uint64_t N = 1ull << L;
    for (uint32_t k = 0; k < 3; k++) cur[k] = k < K ? tables[k] : nullptr;
    for (uint32_t k = 0; k < K; k++) {
        buf[1][k] = L >= 1 ? s->alloc<fr_t>(N >> 1) : nullptr;
        buf[0][k] = L >= 2 ? s->alloc<fr_t>(N >> 2) : nullptr;
    }
    // suffix eq tables over w[t0+1 .. t0+n_eq_loc-1]: LO (pair-summed in the round kernel) x HI (<= 10 vars)
    HI = LO[0] = LO[1] = HP[0] = HP[1] = nullptr;
    // HI variables: 10 for the unfactored kernel (per-pair LO x HI); 5 for the factored K = 2 kernel, whose
    // CTAs apply HI once per group of 2^lo_cnt pairs (groups stay large while LO holds most variables)
    const uint32_t hmax = (factored && K == 2) ? 5 : 10;
    hb = n_eq_loc >= 1 ? (n_eq_loc - 1 < hmax ? n_eq_loc - 1 : hmax) : 0;
    lo0 = n_eq_loc >= 1 ? n_eq_loc - 1 - hb : 0;
    if (n_eq_loc >= 2) {
        HI = s->alloc<fr_t>(1ull << hb);
        eq_table_dev(ctx, d_w + t0 + 1 + lo0, hb, nullptr, HI, *s);
        if (lo0) {
            LO[0] = s->alloc<fr_t>(1ull << lo0);
            LO[1] = s->alloc<fr_t>(1ull << (lo0 - 1));
            eq_table_dev(ctx, d_w + t0 + 1, lo0, nullptr, LO[0], *s);
        }
        HP[0] = s->alloc<fr_t>(1ull << hb);
        HP[1] = s->alloc<fr_t>(1ull << hb);
    }
    lo_level = 0;
    hp_next = 0;
    hi_cur = HI;
    if (!partials) {
        partials = s->alloc<fr_t>((size_t)ctx->num_sms * 4 * 4);
        ticket = s->alloc_zero<unsigned int>(1);
    }
}

void ScEngine::set_i32(const int32_t* const src[3]) {
    // the factored K = 2 kernels take round 0 from int32 tables only when both are int32: one int32 table
    // next to an Fr table (the rescale's W and aux, D26) is embedded here like the other paths
    const bool fused = factored && K == 2 && ((src[0] != nullptr) == (src[1] != nullptr));
    for (uint32_t k = 0; k < K; k++) {
        i32[k] = src[k];
        if (src[k] && !fused)
            embed_i32_dev(ctx, src[k], 1ull << L, const_cast<fr_t*>(cur[k]));
    }
    if (!fused)
        for (uint32_t k = 0; k < 3; k++) i32[k] = nullptr;
}

void ScEngine::materialize() {
    const uint32_t tl = t - t0;
    if (!(tl == 0 || (tl == 1 && int0_used))) return;
    for (uint32_t k = 0; k < K; k++)
        if (i32[k]) embed_i32_dev(ctx, i32[k], 1ull << L, const_cast<fr_t*>(cur[k]));
    for (uint32_t k = 0; k < 3; k++) i32[k] = nullptr;
    int0_used = false;
}

void ScEngine::round(fr_t* part_out) {
    const uint32_t tl = t - t0;
    ZK_REQUIRE(tl < L, ZK_ERR_INTERNAL, "sumcheck engine: no rounds left");
    ScRoundArgs a;
    memset(&a, 0, sizeof a);
    const bool fold = tl > 0;
    const uint64_t n_pairs = 1ull << (L - tl - 1);
    for (uint32_t k = 0; k < K; k++) {
        a.src[k] = cur[k];
        a.dst[k] = fold ? buf[tl & 1][k] : nullptr;
    }
    a.n_pairs = n_pairs;
    a.r_prev = fold ? d_r + (t - 1) : nullptr;
    const uint32_t n_eq_end = t0 + n_eq_loc;
    if (t < n_eq_end && n_eq_end - t - 1 >= 1) {
        const uint32_t nv = n_eq_end - t - 1;
        const uint32_t lo_cnt = nv > hb ? nv - hb : 0;
        if (lo_cnt >= 1) {
            a.eq_mode = 1;
            a.eq_cur = LO[lo_level];
            a.eq_hi = HI;
            a.eq_next = LO[lo_level ^ 1];
            a.lo_cnt = lo_cnt;
            a.hb = hb;
        } else {
            a.eq_mode = 2;
            a.eq_cur = hi_cur;
            a.eq_next = HP[hp_next];
            a.lo_cnt = nv;
        }
    }
    a.partials = partials;
    a.ticket = ticket;
    a.st = tr->d_st;
    a.t = t;
    a.n_eq = n_eq;
    a.w = d_w;
    a.claim = d_claim;
    a.compute_claim = (t == 0 && !claim_given) ? 1 : 0;
    a.claim_bytes = d_proof + 12;
    a.msg_out = d_proof + 44 + 32ull * t * nev();
    a.r_out = d_r + t;
    a.point_out = d_point + 32ull * t;
    a.part_out = part_out;
    a.scale = d_scale;
    const bool der = derive && fold && !part_out && K == 2 && factored && !zero;
    if (derive && !part_out) {
        a.run_claim = run_claim;
        a.winv = winv;
    }
    if (der && tl == 1 && winv) ZK_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->aux_ev[1], 0));   // w^-1 ready
    if (zero) {
        const unsigned int grid = grid_for(ctx, n_pairs, 256, 4);
        if (fold)
            ZK_LAUNCH(ctx, k_sc_zero_round<true>, grid, 256, 0, a);
        else
            ZK_LAUNCH(ctx, k_sc_zero_round<false>, grid, 256, 0, a);
    } else if (K == 2 && factored) {
        Sc2Args A;
        memset(&A, 0, sizeof A);
        A.r = a;
        const bool from_i32 = tl == 0 && (i32[0] || i32[1]);
        if (from_i32) ZK_REQUIRE(i32[0] && i32[1], ZK_ERR_INTERNAL, "sumcheck: mixed int32 / Fr tables in round 0");
        // work items: (group of pairs sharing one HI value) x slices, at most two waves of 2 CTAs per SM
        const uint32_t glog = a.eq_mode ? a.lo_cnt : 0;
        const uint64_t ngroups = a.eq_mode ? ((n_pairs >> glog) ? (n_pairs >> glog) : 1) : 1;
        const uint64_t gsize = a.eq_mode ? (n_pairs < (1ull << glog) ? n_pairs : (1ull << glog)) : n_pairs;
        const uint64_t cap = (uint64_t)ctx->num_sms * 2;
        A.flat = a.eq_mode && gsize < 1024;   // small groups: per-pair HI product instead
        const uint64_t ng = A.flat ? 1 : ngroups, gs = A.flat ? n_pairs : gsize;
        // slices: enough items to fill the grid (one pair per thread at least), ~8 items per CTA when
        // the round is large (static round robin stays balanced), never below 256 pairs per item
        const uint64_t want = (n_pairs + 255) / 256 < cap ? (n_pairs + 255) / 256 : cap;
        uint64_t slices = 1;
        while (gs / (slices * 2) >= 256 && (ng * slices < want || (ng * slices * 2 <= 8 * cap && gs / (slices * 2) >= 2048)))
            slices *= 2;
        A.slices = (uint32_t)slices;
        const unsigned int grid = (unsigned int)(ng * slices < cap ? ng * slices : cap);
        // int32 round 0 in exact integers (grouped eq weights only; ZKDL_SC_INT0=0 disables it)
        static const bool int0_off = getenv("ZKDL_SC_INT0") && atoi(getenv("ZKDL_SC_INT0")) == 0;
        const bool int0 = from_i32 && a.eq_mode != 0 && !A.flat && !int0_off;
        if (from_i32 || (tl == 1 && int0_used))
            for (int k = 0; k < 2; k++) {
                A.i32[k] = i32[k];
                A.emb[k] = const_cast<fr_t*>(cur[k]);
            }
        if (int0) {
            ZK_LAUNCH(ctx, k_sc_round0_int, grid, 256, 0, A);
            int0_used = true;
        } else if (from_i32) {
            ZK_LAUNCH(ctx, k_sc_round2f<2>, grid, 256, 0, A);
        } else if (fold && tl == 1 && int0_used) {
            if (der)
                ZK_LAUNCH(ctx, k_sc_round2f<7>, grid, 256, 0, A);
            else
                ZK_LAUNCH(ctx, k_sc_round2f<3>, grid, 256, 0, A);
        } else if (fold) {
            if (der)
                ZK_LAUNCH(ctx, k_sc_round2f<5>, grid, 256, 0, A);
            else
                ZK_LAUNCH(ctx, k_sc_round2f<1>, grid, 256, 0, A);
        } else {
            ZK_LAUNCH(ctx, k_sc_round2f<0>, grid, 256, 0, A);
        }
    } else {
        unsigned int grid = grid_for(ctx, n_pairs, 256, 4);
        if (K == 1) launch_round<1>(ctx, fold, grid, a);
        else if (K == 2) launch_round<2>(ctx, fold, grid, a);
        else launch_round<3>(ctx, fold, grid, a);
    }
    if (a.eq_mode == 1) {
        lo_level ^= 1;
    } else if (a.eq_mode == 2) {
        hi_cur = HP[hp_next];
        hp_next ^= 1;
    }
    if (fold)
        for (uint32_t k = 0; k < K; k++) cur[k] = buf[tl & 1][k];
    t++;
}

void ScEngine::combine(const fr_t* all, uint32_t G) {
    ZK_LAUNCH(ctx, k_sc_combine, 1, 32, 0, all, G, (int)K, t - 1, n_eq, d_w, d_claim, (t - 1 == 0 && !claim_given) ? 1 : 0,
              tr->d_st, d_proof + 12, d_proof + 44 + 32ull * (t - 1) * (K + 1), d_r + (t - 1), d_point + 32ull * (t - 1));
}

void ScEngine::header() {
    uint8_t hdr[12];
    const uint32_t hv[3] = {m, n_eq, K};
    for (int i = 0; i < 3; i++)
        for (int k = 0; k < 4; k++) hdr[4 * i + k] = (uint8_t)(hv[i] >> (8 * k));
    ZK_LAUNCH(ctx, k_sc_header, 1, 32, 0, tr->d_st, make_bytes(hdr, 12), d_claim, claim_given ? 1 : 0, d_proof + 12);
}

void ScEngine::finals() {
    ZK_LAUNCH(ctx, k_sc_finals, 1, 32, 0, cur[0], K > 1 ? cur[1] : cur[0], K > 2 ? cur[2] : cur[0], (int)K, d_r + (m - 1),
              tr->d_st, d_proof + 44 + 32ull * m * nev(), d_finals);
}

// ---------------------------------------------------------------- persistent small-statement prover
// Every round of a small statement (2^m <= 2^SC_ALL_MAX_LOG entries) in ONE cooperative launch: the
// per-round kernel launch, the cold re-fetch of the round code and the separate finalizer launch are
// replaced by two device-side waits per round (blocks publish partials and bump a monotonic arrival
// counter; block 0 reduces them, runs the transcript step on its warp 0 and publishes r_t through a
// round flag).  Eq suffix levels E_t = beta(w_{t+1..n_eq-1}, .) are pair-summed one level ahead.
constexpr uint32_t SC_ALL_MAX_LOG = 18;
constexpr uint64_t SC_SOLO_PAIRS = 512;   // rounds with at most this many pairs: the reducer block alone

struct ScAllArgs {
    const fr_t* src[3];
    fr_t* buf[2][3];
    fr_t* E[2];                 // E[0] = level 0 = beta(w_1..w_{n_eq-1}); levels alternate
    uint32_t m, n_eq;
    const fr_t* w;
    fr_t* claim;
    int compute_claim;
    uint8_t* st;
    uint8_t* proof;
    fr_t* d_r;
    uint8_t* d_point;
    fr_t* d_finals;
    fr_t* partials;             // gridDim.x * 4
    unsigned int* arrive;       // monotonic: blocks that finished round t = (t+1) * gridDim.x
    unsigned int* flag;         // rounds whose challenge is published
    const fr_t* r_first;        // continuation of a larger statement: round 0 folds by this challenge
    unsigned long long* trace;  // diagnostics (ZKDL_SCALL_TRACE): 4 timestamps per round (block 0), or null
};

__device__ __forceinline__ unsigned long long sc_globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned int ld_volatile(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int K>
__global__ void __launch_bounds__(256) k_sc_all(ScAllArgs a) {
    __shared__ fr_t sm_red[32 * (K + 1)];
    __shared__ fr_t tot[K + 1];
    __shared__ FsScratch fs;
    __shared__ fr_t claim_sm;
    const uint32_t m = a.m, n_eq = a.n_eq;
    const int tid = threadIdx.x;
    if (blockIdx.x == 0 && tid < 32) fs_begin(fs, a.st);
    const long long c_start = clock64();
    const unsigned long long g_start = a.trace ? sc_globaltimer() : 0ull;
    for (uint32_t t = 0; t < m; t++) {
        const uint64_t n_pairs = 1ull << (m - t - 1);
        if (a.trace && blockIdx.x == 0 && tid == 0) a.trace[10 * t] = sc_globaltimer();
        // the last rounds (<= SC_SOLO_PAIRS pairs) run on the reducer block alone: no partials, arrival
        // counter or round flag, one __syncthreads per round (the workers' last folds are visible: they
        // fenced before their final arrival, which block 0 waited for)
        const bool solo = gridDim.x == 1 || n_pairs <= SC_SOLO_PAIRS;
        if (solo && blockIdx.x != 0) return;
        const bool fold0 = a.r_first != nullptr;
        const bool folding = t > 0 || fold0;
        const fr_t* src[K];
        fr_t* dst[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            src[k] = (t == 0 || (t == 1 && !fold0)) ? a.src[k] : a.buf[(t - 1) & 1][k];
            dst[k] = a.buf[t & 1][k];
        }
        fr_t r;
        if (folding) {
            const uint4* q = reinterpret_cast<const uint4*>(t > 0 ? &a.d_r[t - 1] : a.r_first);
            uint4 x = __ldcg(q), y = __ldcg(q + 1);
            r = fr_t{{x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w}};
        }
        const bool has_e = n_eq >= 2 && t + 1 < n_eq;
        const uint32_t nv = has_e ? n_eq - t - 1 : 0;
        const fr_t* Ecur = a.E[t & 1];
        fr_t* Enext = a.E[(t + 1) & 1];
        const uint64_t emask = (1ull << nv) - 1, enext = nv >= 1 ? (1ull << (nv - 1)) : 0;
        fr_t acc[K + 1];
#pragma unroll
        for (int x = 0; x <= K; x++) acc[x] = fr_zero();
        const uint64_t nworkers = gridDim.x - 1;
        const uint64_t b0 = solo ? (uint64_t)tid : (blockIdx.x == 0 ? n_pairs : (blockIdx.x - 1) * (uint64_t)blockDim.x + tid);
        const uint64_t bs = solo ? (uint64_t)blockDim.x : nworkers * blockDim.x;
        for (uint64_t b = b0; b < n_pairs; b += bs) {
            fr_t lo[K], d[K];
            // out-of-line product bodies: the kernel's code stays inside the instruction cache (the inlined
            // products made k_sc_all ~290 KB of SASS, every round re-fetched from L2); K = 2 groups its
            // independent products in pairs / triples (shorter per-pair latency in the small rounds)
            if (K == 2 && folding) {
                const fr_t* s0 = src[0] + 4 * b;
                const fr_t* s1 = src[K - 1] + 4 * b;
                const fr_t x0 = fr_load_l2(s0), x1 = fr_load_l2(s0 + 1), x2 = fr_load_l2(s0 + 2), x3 = fr_load_l2(s0 + 3);
                const fr_t y0 = fr_load_l2(s1), y1 = fr_load_l2(s1 + 1), y2 = fr_load_l2(s1 + 2), y3 = fr_load_l2(s1 + 3);
                const fr2p_t f = fr_mul2_ni(r, fr_sub(x1, x0), r, fr_sub(x3, x2));
                const fr2p_t g = fr_mul2_ni(r, fr_sub(y1, y0), r, fr_sub(y3, y2));
                const fr_t v0 = fr_add(x0, f.x), v1 = fr_add(x2, f.y), w0 = fr_add(y0, g.x), w1 = fr_add(y2, g.y);
                fr_store(dst[0] + 2 * b, v0);
                fr_store(dst[0] + 2 * b + 1, v1);
                fr_store(dst[K - 1] + 2 * b, w0);
                fr_store(dst[K - 1] + 2 * b + 1, w1);
                lo[0] = v0;
                d[0] = fr_sub(v1, v0);
                lo[K - 1] = w0;
                d[K - 1] = fr_sub(w1, w0);
            } else
#pragma unroll
            for (int k = 0; k < K; k++) {
                fr_t v0, v1;
                if (folding) {
                    const fr_t* s = src[k] + 4 * b;
                    fr_t x0 = fr_load_l2(s), x1 = fr_load_l2(s + 1), x2 = fr_load_l2(s + 2), x3 = fr_load_l2(s + 3);
                    v0 = fr_add(x0, fr_mul_ni(r, fr_sub(x1, x0)));
                    v1 = fr_add(x2, fr_mul_ni(r, fr_sub(x3, x2)));
                    fr_store(dst[k] + 2 * b, v0);
                    fr_store(dst[k] + 2 * b + 1, v1);
                } else {
                    v0 = fr_load_l2(src[k] + 2 * b);
                    v1 = fr_load_l2(src[k] + 2 * b + 1);
                }
                lo[k] = v0;
                d[k] = fr_sub(v1, v0);
            }
            fr_t e;
            if (has_e) {
                const uint4* q = reinterpret_cast<const uint4*>(&Ecur[b & emask]);
                uint4 x = __ldcg(q), y = __ldcg(q + 1);
                e = fr_t{{x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w}};
                if (b < enext) {
                    const uint4* q0 = reinterpret_cast<const uint4*>(&Ecur[2 * b]);
                    uint4 a0 = __ldcg(q0), a1 = __ldcg(q0 + 1), b0 = __ldcg(q0 + 2), b1 = __ldcg(q0 + 3);
                    fr_store(&Enext[b], fr_add(fr_t{{a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w}},
                                               fr_t{{b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w}}));
                }
            }
            if (K == 2) {   // the three evaluations (X = 0, 1, 2), then their eq weights, as triples
                const fr_t a1 = fr_add(lo[0], d[0]), b1 = fr_add(lo[K - 1], d[K - 1]);
                const fr3_t p = fr_mul3_ni(lo[0], lo[K - 1], a1, b1, fr_add(a1, d[0]), fr_add(b1, d[K - 1]));
                fr3_t q = p;
                if (has_e) q = fr_mul3_ni(p.x, e, p.y, e, p.z, e);
                acc[0] = fr_add(acc[0], q.x);
                acc[1] = fr_add(acc[1], q.y);
                acc[K] = fr_add(acc[K], q.z);
            } else {
                fr_t v[K];
#pragma unroll
                for (int k = 0; k < K; k++) v[k] = lo[k];
#pragma unroll
                for (int x = 0; x <= K; x++) {
                    fr_t p = v[0];
#pragma unroll
                    for (int k = 1; k < K; k++) p = fr_mul_ni(p, v[k]);
                    if (has_e) p = fr_mul_ni(p, e);
                    acc[x] = fr_add(acc[x], p);
                    if (x < K)
#pragma unroll
                        for (int k = 0; k < K; k++) v[k] = fr_add(v[k], d[k]);
                }
            }
        }
        if (solo) {   // block 0 alone: its own sums are the round totals
            block_reduce_fr_rolled<K + 1>(acc, sm_red);
            if (tid == 0)
#pragma unroll
                for (int x = 0; x <= K; x++) tot[x] = acc[x];
            __syncthreads();
        } else if (blockIdx.x != 0) {   // worker: publish the block partial
            if (a.trace && blockIdx.x == 1 && tid == 0) a.trace[10 * t + 6] = sc_globaltimer();
            block_reduce_fr_rolled<K + 1>(acc, sm_red);
            if (a.trace && blockIdx.x == 1 && tid == 0) a.trace[10 * t + 7] = sc_globaltimer();
            if (tid == 0) {
#pragma unroll
                for (int x = 0; x <= K; x++) fr_store(&a.partials[(blockIdx.x - 1) * (K + 1) + x], acc[x]);
                __threadfence();
                atomicAdd(a.arrive, 1u);
            }
        }
        if (blockIdx.x == 0) {   // dedicated reducer + transcript block (its I-cache keeps only this code)
            if (!solo) {
                if (tid == 0) {
                    while (ld_volatile(a.arrive) < (t + 1) * (gridDim.x - 1)) {
                    }
                    __threadfence();
                    if (a.trace) a.trace[10 * t + 1] = sc_globaltimer();
                }
                __syncthreads();
                fr_t s_[K + 1];
#pragma unroll
                for (int x = 0; x <= K; x++) s_[x] = fr_zero();
                for (unsigned int bb = tid; bb < gridDim.x - 1; bb += blockDim.x)
#pragma unroll
                    for (int x = 0; x <= K; x++) {
                        const uint4* q = reinterpret_cast<const uint4*>(&a.partials[bb * (K + 1) + x]);
                        uint4 xx = __ldcg(q), yy = __ldcg(q + 1);
                        s_[x] = fr_add(s_[x], fr_t{{xx.x, xx.y, xx.z, xx.w, yy.x, yy.y, yy.z, yy.w}});
                    }
                block_reduce_fr_rolled<K + 1>(s_, sm_red);
                if (tid == 0)
#pragma unroll
                    for (int x = 0; x <= K; x++) tot[x] = s_[x];
                __syncthreads();
            }
            if (a.trace && tid == 0) a.trace[10 * t + 2] = sc_globaltimer();
            if (tid < 32) {
                const int lane = tid;
                if (t == 0 && a.compute_claim) {
                    if (lane == 0) {
                        fr_t c;
                        if (n_eq >= 1) {
                            fr_t w0 = fr_load(&a.w[0]);
                            c = fr_add(fr_mul_cold(fr_sub(fr_one(), w0), tot[0]), fr_mul_cold(w0, tot[1]));
                        } else {
                            c = fr_add(tot[0], tot[1]);
                        }
                        fr_store(a.claim, c);
                        claim_sm = c;
                    }
                    __syncwarp();
                    fs_absorb_frs(fs, "sc/claim", claim_sm, 1, a.proof + 12);
                }
                const long long ca = clock64();
                fs_absorb_frs(fs, "sc/msg", lane <= K ? tot[lane & 3] : fr_zero(), K + 1, a.proof + 44 + 32ull * t * (K + 1));
                const long long cb = clock64();
                if (a.trace && lane == 0) a.trace[10 * t + 3] = sc_globaltimer();
                fr_t rt = fs_challenge(fs, "sc/r");
                const long long cc = clock64();
                if (a.trace && lane == 0) {
                    a.trace[10 * t + 4] = sc_globaltimer();
                    a.trace[10 * t + 8] = (unsigned long long)(cb - ca);
                    a.trace[10 * t + 9] = (unsigned long long)(cc - cb);
                }
                if (lane == 0) {
                    fr_store(&a.d_r[t], rt);
                    fr_canon_to_bytes(fs.rc, a.d_point + 32ull * t);
                    __threadfence();
                    if (!solo) atomicExch(a.flag, t + 1);
                    if (a.trace) a.trace[10 * t + 5] = sc_globaltimer();
                }
            }
        } else {
            if (tid == 0) {
                // back off while the reducer hashes: the waiting warps leave the issue slots to
                // kernels of the other stream sharing the SM
                while (ld_volatile(a.flag) < t + 1) __nanosleep(256);
                __threadfence();
            }
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && tid < 32) {   // finals on the last 2-element tables
        const int lane = tid;
        const fr_t* T = lane == 0 ? a.buf[(m - 1) & 1][0] : (lane == 1 ? a.buf[(m - 1) & 1][K > 1 ? 1 : 0]
                                                                        : a.buf[(m - 1) & 1][K > 2 ? 2 : 0]);
        if (m == 1 && !a.r_first) T = lane == 0 ? a.src[0] : (lane == 1 ? a.src[K > 1 ? 1 : 0] : a.src[K > 2 ? 2 : 0]);
        fr_t f = fr_zero();
        if (lane < K) {
            fr_t rr = fr_load(&a.d_r[m - 1]);
            fr_t x0 = fr_load_l2(T), x1 = fr_load_l2(T + 1);
            f = fr_add(x0, fr_mul_cold(rr, fr_sub(x1, x0)));
            if (a.d_finals) fr_store(&a.d_finals[lane], f);
        }
        fs_absorb_frs(fs, "sc/final", f, K, a.proof + 44 + 32ull * m * (K + 1));
        fs_end(fs, a.st);
        if (a.trace && lane == 0) {   // SM clock of the reducer block over the launch
            a.trace[10ull * m] = (unsigned long long)(clock64() - c_start);
            a.trace[10ull * m + 1] = sc_globaltimer() - g_start;
        }
    }
}

// CTA size of the persistent small-statement prover (ZKDL_SCALL_T=128 for experiments: measured no
// better in the C4 window, 11.80 vs 11.65 ms)
static int sc_all_threads() {
    const char* e = getenv("ZKDL_SCALL_T");
    return (e && atoi(e) == 128) ? 128 : 256;
}

template <int K>
static void launch_all(zk_ctx* ctx, const ScAllArgs& a, unsigned int grid) {
    void* args[] = {(void*)&a};
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    const bool prof = ctx->prof_match("k_sc_all");
    if (prof) {
        ev_a = ctx->take_event();
        ev_b = ctx->take_event();
        cudaEventRecord(ev_a, ctx->stream);
    }
    ZK_CUDA(cudaLaunchCooperativeKernel((const void*)k_sc_all<K>, dim3(grid), dim3(sc_all_threads()), args, 0, ctx->stream));
    after_launch(ctx, "k_sc_all");
    if (prof) {
        cudaEventRecord(ev_b, ctx->stream);
        ctx->recs.push_back({"k_sc_all", ev_a, ev_b});
    }
}

template <int K>
static unsigned int all_grid(zk_ctx* ctx, uint32_t m) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sc_all<K>, sc_all_threads(), 0);
    if (per_sm < 1) per_sm = 1;
    // at most one block per SM: the rounds are latency-bound after the first few, and a persistent
    // grid that fills the GPU would crowd out the zkReLU kernels running on the other stream
    uint64_t cap = (uint64_t)per_sm * ctx->num_sms;
    if (cap > (uint64_t)ctx->num_sms) cap = (uint64_t)ctx->num_sms;
    if (ctx->sm_budget > 0 && cap > (uint64_t)ctx->sm_budget) cap = (uint64_t)ctx->sm_budget;
    if (cap < 2) cap = 2;   // one worker + the reducer block
    const uint64_t T = (uint64_t)sc_all_threads();
    uint64_t need = ((1ull << (m - 1)) + T - 1) / T + 1;   // + the reducer block
    if (need < 2) need = 2;
    return (unsigned int)(need < cap ? need : cap);
}

static void sumcheck_prove_small(zk_ctx* ctx, zk_transcript* tr, const ScStatement& S, Scratch& s) {
    const uint32_t m = S.m, n_eq = S.n_eq, K = S.K;
    uint8_t hdr[12];
    const uint32_t hv[3] = {m, n_eq, K};
    for (int i = 0; i < 3; i++)
        for (int k = 0; k < 4; k++) hdr[4 * i + k] = (uint8_t)(hv[i] >> (8 * k));
    ZK_LAUNCH(ctx, k_sc_header, 1, 32, 0, tr->d_st, make_bytes(hdr, 12), S.d_claim, S.claim_given ? 1 : 0, S.d_proof + 12);
    ScAllArgs a;
    memset(&a, 0, sizeof a);
    const uint64_t N = 1ull << m;
    for (uint32_t k = 0; k < K; k++) {
        a.src[k] = S.tables[k];
        a.buf[1][k] = s.alloc<fr_t>(N >> 1);
        a.buf[0][k] = s.alloc<fr_t>(m >= 2 ? N >> 2 : 1);
    }
    if (n_eq >= 2) {
        a.E[0] = s.alloc<fr_t>(1ull << (n_eq - 1));
        a.E[1] = s.alloc<fr_t>(n_eq >= 3 ? 1ull << (n_eq - 2) : 1);
        eq_table_dev(ctx, S.d_w + 1, n_eq - 1, nullptr, a.E[0], s);
    }
    a.m = m;
    a.n_eq = n_eq;
    a.w = S.d_w;
    a.claim = S.d_claim;
    a.compute_claim = S.claim_given ? 0 : 1;
    a.st = tr->d_st;
    a.proof = S.d_proof;
    a.d_r = S.d_r;
    a.d_point = S.d_point;
    a.d_finals = S.d_finals;
    unsigned int grid = K == 1 ? all_grid<1>(ctx, m) : K == 2 ? all_grid<2>(ctx, m) : all_grid<3>(ctx, m);
    a.partials = s.alloc<fr_t>((size_t)grid * 4);
    unsigned int* ctr = s.alloc_zero<unsigned int>(2);
    a.arrive = ctr;
    a.flag = ctr + 1;
    static const bool trace = getenv("ZKDL_SCALL_TRACE") != nullptr;
    if (trace) a.trace = s.alloc_zero<unsigned long long>(10ull * m + 2);
    if (K == 1) launch_all<1>(ctx, a, grid);
    else if (K == 2) launch_all<2>(ctx, a, grid);
    else launch_all<3>(ctx, a, grid);
    if (trace) {
        std::vector<unsigned long long> h(10ull * m + 2);
        ZK_CUDA(cudaMemcpyAsync(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
        ZK_CUDA(cudaStreamSynchronize(ctx->stream));
        for (uint32_t t = 0; t < m; t++) {
            const unsigned long long* q = &h[10ull * t];
            const unsigned long long nx = t + 1 < m ? h[10ull * (t + 1)] : q[5];
            auto us = [](unsigned long long a, unsigned long long b) { return a && b ? ((long long)b - (long long)a) / 1e3 : 0.0; };
            fprintf(stderr, "sc_all m=%u grid=%u t=%u arrive %.1f us, reduce %.1f, absorb %.1f, challenge %.1f, publish %.1f, "
                    "next %.1f | worker1 compute done %.1f, block reduce %.1f | absorb %llu cycles, challenge %llu\n", m, grid, t, us(q[0], q[1]),
                    q[1] ? us(q[1], q[2]) : us(q[0], q[2]), us(q[2], q[3]), us(q[3], q[4]), us(q[4], q[5]), us(q[5], nx),
                    us(q[0], q[6]), us(q[6], q[7]), q[8], q[9]);
        }
        fprintf(stderr, "sc_all m=%u: reducer block SM clock %.3f GHz\n", m, (double)h[10ull * m] / (double)h[10ull * m + 1]);
    }
}

// out[i] = in[i]^-1 (binary extended Euclid, one value per warp; traps on zero: probability ~2^-250 per transcript
// challenge)
__global__ void k_fr_inv_batch(const fr_t* in, uint32_t n, fr_t* out) {
    const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= n || (threadIdx.x & 31)) return;
    const fr_t x = fr_load(&in[i]);
    if (fr_is_zero(x)) __trap();
    fr_store(&out[i], fr_inv_bgcd(x));
}

void sumcheck_prove_dev(zk_ctx* ctx, zk_transcript* tr, const ScStatement& S, Scratch& s) {
    const uint32_t m = S.m, n_eq = S.n_eq, K = S.K;
    ZK_REQUIRE(m >= 1 && m <= 40 && n_eq <= m && K >= 1 && K <= 3, ZK_ERR_ARG, "sumcheck: bad m / n_eq / K");
    if (m <= SC_ALL_MAX_LOG && !getenv("ZKDL_NO_PERSISTENT") && !ctx->no_persist) {
        for (uint32_t k = 0; k < K; k++)
            if (S.i32[k]) embed_i32_dev(ctx, S.i32[k], 1ull << m, const_cast<fr_t*>(S.tables[k]));
        sumcheck_prove_small(ctx, tr, S, s);
        return;
    }
    ScEngine e;
    e.ctx = ctx;
    e.tr = tr;
    e.s = &s;
    e.m = m;
    e.n_eq = n_eq;
    e.K = K;
    e.d_w = S.d_w;
    e.d_scale = nullptr;
    e.d_proof = S.d_proof;
    e.d_r = S.d_r;
    e.d_point = S.d_point;
    e.d_claim = S.d_claim;
    e.claim_given = S.claim_given;
    e.d_finals = S.d_finals;
    e.header();
    e.setup(S.tables, m, 0, n_eq);
    e.set_i32(S.i32);
    // derived X = 1 in the folding rounds of the factored K = 2 kernel (ZKDL_SC_DERIVE=0: explicit f(1))
    static const bool der_off = getenv("ZKDL_SC_DERIVE") && atoi(getenv("ZKDL_SC_DERIVE")) == 0;
    if (!der_off && K == 2 && e.factored && m >= 2) {
        e.derive = true;
        e.run_claim = s.alloc<fr_t>(1);
        if (n_eq) {
            e.winv = s.alloc<fr_t>(n_eq);
            cudaStream_t aux = ctx->aux_stream();
            ZK_CUDA(cudaEventRecord(ctx->aux_ev[0], ctx->stream));
            ZK_CUDA(cudaStreamWaitEvent(aux, ctx->aux_ev[0], 0));
            k_fr_inv_batch<<<(n_eq + 3) / 4, 128, 0, aux>>>(S.d_w, n_eq, e.winv);
            after_launch(ctx, "k_fr_inv_batch");
            ZK_CUDA(cudaEventRecord(ctx->aux_ev[1], aux));
        }
    }
    e.run_to_end();
}

constexpr uint32_t SC_TAIL_LOG = 16;

void ScEngine::run_to_end() {
    const bool persistent_ok = !getenv("ZKDL_NO_PERSISTENT") && !ctx->no_persist && !zero;
    while (t < t0 + L) {
        const uint32_t tl = t - t0;
        if (tl >= 1 && persistent_ok && L - tl <= SC_TAIL_LOG) {
            persist_rest();
            return;
        }
        round(nullptr);
    }
    finals();
}

// The remaining local rounds tl .. L-1 (tl >= 1: the tables still need the fold by r_{t-1}) as a
// continuation statement of k_sc_all: m' = L - tl variables, eq over the remaining eq variables, the
// same transcript, proof offsets shifted by t rounds; k_sc_all also writes the finals.
void ScEngine::persist_rest() {
    const uint32_t tl = t - t0, mr = L - tl;
    ZK_REQUIRE(tl >= 1 && mr >= 1, ZK_ERR_INTERNAL, "sumcheck continuation: bad round");
    materialize();
    ScAllArgs a;
    memset(&a, 0, sizeof a);
    for (uint32_t k = 0; k < K; k++) {
        a.src[k] = cur[k];
        a.buf[0][k] = s->alloc<fr_t>(1ull << mr);
        a.buf[1][k] = s->alloc<fr_t>(mr >= 2 ? 1ull << (mr - 1) : 1);
    }
    const uint32_t n_eq_end = t0 + n_eq_loc;
    const uint32_t n_rem = t < n_eq_end ? n_eq_end - t : 0;
    if (n_rem >= 2) {
        a.E[0] = s->alloc<fr_t>(1ull << (n_rem - 1));
        a.E[1] = s->alloc<fr_t>(n_rem >= 3 ? 1ull << (n_rem - 2) : 1);
        eq_table_dev(ctx, d_w + t + 1, n_rem - 1, nullptr, a.E[0], *s);
    }
    a.m = mr;
    a.n_eq = n_rem;
    a.w = d_w + t;
    a.claim = d_claim;
    a.compute_claim = 0;
    a.st = tr->d_st;
    a.proof = d_proof + 32ull * t * (K + 1);   // message of local round i at d_proof + 44 + 32 (t + i)(K + 1)
    a.d_r = d_r + t;
    a.d_point = d_point + 32ull * t;
    a.d_finals = d_finals;
    a.r_first = d_r + t - 1;
    unsigned int grid = K == 1 ? all_grid<1>(ctx, mr) : K == 2 ? all_grid<2>(ctx, mr) : all_grid<3>(ctx, mr);
    a.partials = s->alloc<fr_t>((size_t)grid * 4);
    unsigned int* ctr = s->alloc_zero<unsigned int>(2);
    a.arrive = ctr;
    a.flag = ctr + 1;
    if (K == 1) launch_all<1>(ctx, a, grid);
    else if (K == 2) launch_all<2>(ctx, a, grid);
    else launch_all<3>(ctx, a, grid);
    t = t0 + L;
}

uint64_t sumcheck_proof_len(uint32_t m, uint32_t K) { return 12 + 32 + 32ull * m * (K + 1) + 32ull * K; }

}  // namespace zk
