// gram.cu — zkReLU bit sums on the 5th-generation tensor cores (row a8, j-phase inputs).
//
// The j-rounds of the zkReLU sumcheck (relu.cu) need, for the bit words w_s(i) (s = 0: Z, s = 1: G_A,
// masked to Q+R bits) and eq weights c_x(i) = eq(u_x, i):
//     M_x[j]       = sum_i c_x(i) [1 - sig_i]^{x in {A, G_Z}} bit_j(w_{s(x)}(i))        (linear cells)
//     C_s[j1][j2]  = sum_i e_b(i) bit_j1(w_s(i)) bit_j2(w_s(i)),   j1 <= j2              (Gram cells)
// (P:L449-470 AIVP with the bits-first order of DESIGN.md D5/D12).  Both are dense contractions over i:
// with the eq table split eq(u, i) = LO(i mod 2^16) HI(i >> 16) and the LO values (R^2-scaled residues)
// written as 32 bytes L_k, a row segment of entries gives exact int32 sums
//     G_k[j1][j2] = sum_i L_k(i) b_j1(i) b_j2(i)          (A = L_k & b_j1 : u8,  B = b_j2 : u8)
// which tcgen05.mma.kind::i8 computes with A in TMEM (rows (j1, k): 4 j1 x 32 limbs per M = 128 tile),
// B in shared memory (32 bit planes x 32 entries per K step) and the s32 accumulators in TMEM.  At the
// end of a row segment the 32 limb sums of a cell are recombined, sum_k 2^{8k} G_k (< p 2^24),
// Montgomery-reduced and multiplied by HI[row].
//
// Round 0 of the i-phase from the same pass (round 2): the K steps of a 64-entry group take its 32 even
// entries, then its 32 odd ones (the Gram sums do not depend on the order), and the linear cells are kept
// per parity over PAIRS b with the eq tables E'_x = eq(u_x[1..], b) (variable 0 of i pulled out):
//     Lin[s][par][q][j] = sum_b E'_x(b) g_q(b) bit_j(w_s(2b + par)),  g_0 = 1, g_1 = o(2b + par), g_2 = o(2b + 1 - par)
// (o = 1 - sig of the Z word).  M_x = beta(u_x[0], 0) Lin[..][0][q] + beta(u_x[0], 1) Lin[..][1][q] (q < 2) are the
// j-phase cells as before, and after the j-rounds the first i-round's linear terms T_a(0), T_c(0), T_c(inf)
// follow from Lin without touching the entries again (k_relu_jrounds; the round kernel then sums the
// binary-check terms only).  C_s is symmetric: the tiles with j1 >= 16 only need j2 >= 16 (N = 16 MMAs).
// CTA roles: blockIdx.x = 2 g + s: word s, K-step range g of G.  Warps 0-7 produce the operands
// (warp w: bit planes 4w..4w+3; C tiles t = 4 (w / 4) .. +3 with j1 = 4t + (w % 4); warps 0, 1 also the
// linear-cell tile), warp 8 issues the MMAs.  TMEM columns: [0, 256) Gram accumulators (tile t at 32t),
// [256, 288) linear-cell accumulator, [288, 504) three A stages of 9 tiles x 8 columns.
#include "relu.cuh"
#include "tables.cuh"
#include "tc.cuh"

namespace zk {

// GR_SYM = 0 (A/B build): every Gram tile N = 32 (the full 32 x 32 cells), two A stages to fit TMEM
#ifndef GR_SYM
#define GR_SYM 1
#endif
// GR_SELFGATE = 1 (A/B build, measured slower: the Gram 2.12 -> 2.55 ms): the linear-tile rows built by warps 4-6, each gating its own row
// with a ballot of the sign words it loads itself (no shared gate words, nothing added to the barrier's
// critical path); 0: warps 0-2 build the rows, warp GR_GATE_WARP publishes the gates through shared memory
#ifndef GR_SELFGATE
#define GR_SELFGATE 0
#endif
#ifndef GR_GATE_WARP
#define GR_GATE_WARP 7   // builds the sign gates of the linear tile (a warp without linear-tile rows)
#endif
#if GR_SYM
constexpr int GR_STAGES = 3;
constexpr uint32_t GR_ACC_HI = 128;   // tiles t >= 4 (N = 16)
constexpr uint32_t GR_ACC_LIN = 192;  // + 32 par
constexpr uint32_t GR_ASTAGE = 256;
#else
constexpr int GR_STAGES = 2;
constexpr uint32_t GR_ACC_HI = 128;
constexpr uint32_t GR_ACC_LIN = 256;
constexpr uint32_t GR_ASTAGE = 320;
#endif
constexpr uint32_t GR_STAGE_COLS = 72;
// instruction descriptors, kind::i8: D s32 (bits 4-5 = 2), A and B u8, both K-major, N (N >> 3 at bit 17),
// M = 128 (M >> 4 at bit 24)
constexpr uint32_t GR_IDESC = (2u << 4) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t GR_IDESC16 = (2u << 4) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

// Operand chunks (256 entries = 8 K steps) are streamed into shared memory by a loader warp with bulk
// async copies: the bit words and, per eq table used, 32 limb rows of 256 bytes padded to 272 (so the
// 32 lanes' 32-byte reads of one K step fall in distinct bank groups).
constexpr int GR_CH_KS = 8;
constexpr int GR_CH = 32 * GR_CH_KS;
constexpr int GR_LROW = GR_CH + 16;
constexpr int GR_LBLK = 32 * GR_LROW;   // one chunk of one limb-transposed table
constexpr int GR_PCH = GR_CH / 2;       // pairs per chunk
constexpr int GR_PROW = GR_PCH + 16;
constexpr int GR_PBLK = 32 * GR_PROW;   // one chunk of one limb-transposed pair table
constexpr int GR_CSTAGES = 3;

struct GramArgs {
    const int32_t* Z;
    const int32_t* GA;
    uint64_t nch;          // chunks (D / 256)
    uint32_t ch_per_row;   // 2^lo_bits / 256
    uint32_t qr_mask, sig_bit, B;
    const uint8_t* LOTb;   // e_b's LO table limb-transposed, entries in K-step order (k_lo_limbs_perm): chunk c
                           // of a row at LOTb + c * GR_LBLK, [limb k][GR_LROW]
    const uint8_t* LOTp[4];// E'_x's LO tables over pairs (x = Z, A, GA, GZ), chunk c at + c * GR_PBLK: [limb][GR_PROW]
    const fr_t* HI[5];
    uint32_t G;            // CTAs per word
    fr_t* partials;        // [2][G][ncs]: ncs = 6B linear cells of the word ([par][q][j]), then its B(B+1)/2 Gram cells
};

struct GramChunk {
    uint32_t z[GR_CH];             // Z words (sign bits; the bit word when s = 0)
    uint32_t w[GR_CH];             // G_A words (s = 1)
    uint8_t lotb[GR_LBLK];         // e_b limb rows (K-step order)
    uint8_t lotp[2][GR_PBLK];      // the word's two linear-cell tables (pairs)
};

struct GramSmem {
    GramChunk ch[GR_CSTAGES];
    uint8_t sB[GR_STAGES][1024];   // B tiles: plane j, entry byte kb at (j/8)*256 + (kb/16)*128 + (j%8)*16 + kb%16
    uint32_t mask[2][32][8];       // plane masks (0xFF bytes) for the K step of parity it & 1
    uint32_t gate[2][8];           // (1 - sig) masks of the K step's entries
    uint32_t gate2[2][8];          // (1 - sig) masks of their pair partners (the other parity)
    uint32_t stage[8][32][33];     // epilogue: warp, column, limb
    fr_t tot[192 + 528];           // running cell totals of this CTA
    uint64_t full[GR_STAGES], empty[GR_STAGES], accfull, cfull[GR_CSTAGES], cempty[GR_CSTAGES];
    uint32_t tmem;
};

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&w)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr), "r"(w[0]),
                 "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                 : "memory");
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t accumulate,
                                       uint32_t idesc = GR_IDESC) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// 4 bits -> 4 bytes of 0x00 / 0xFF
__device__ __forceinline__ uint32_t expand4(uint32_t n) { return ((n * 0x00204081u) & 0x01010101u) * 0xFFu; }

// sum_k 2^{8k} x_k (x_k < 2^25) as a 10-limb integer, Montgomery-reduced
__device__ __forceinline__ fr_t compose_limbs(const uint32_t* x /* 32 limbs, stride 1 */) {
    uint64_t a[9];
#pragma unroll
    for (int i = 0; i < 9; i++) a[i] = 0;
#pragma unroll
    for (int k = 0; k < 32; k++) a[k >> 2] += (uint64_t)x[k] << (8 * (k & 3));
    uint32_t w[10];
    uint64_t c = 0;
#pragma unroll
    for (int i = 0; i < 9; i++) {
        const uint64_t t = a[i] + c;
        w[i] = (uint32_t)t;
        c = t >> 32;
    }
    w[9] = (uint32_t)c;
    return fr_redc_wide(w);
}

__device__ __forceinline__ int gr_tri(int j1, int j2, int B) { return j1 * B - j1 * (j1 - 1) / 2 + (j2 - j1); }

__global__ void __launch_bounds__(320, 1) k_relu_gram(GramArgs a) {
    extern __shared__ __align__(1024) uint8_t gsm_raw[];
    GramSmem& S = *reinterpret_cast<GramSmem*>(gsm_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x & 1;
    const uint32_t g = blockIdx.x >> 1;
    const uint64_t c0 = g * a.nch / a.G, c1 = (g + 1) * a.nch / a.G;   // this CTA's chunks
    const uint32_t B = a.B, T = B * (B + 1) / 2, ncs = 6 * B + T;
    for (uint32_t i = threadIdx.x; i < ncs; i += blockDim.x) S.tot[i] = fr_zero();
    if (warp == 8) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&S.tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        if (lane == 0) {
            for (int i = 0; i < GR_STAGES; i++) {
                mbar_init(&S.full[i], 8);
                mbar_init(&S.empty[i], 1);
            }
            for (int i = 0; i < GR_CSTAGES; i++) {
                mbar_init(&S.cfull[i], 1);
                mbar_init(&S.cempty[i], 8);
            }
            mbar_init(&S.accfull, 1);
            asm volatile("fence.mbarrier_init.release.cluster;");
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem;

    if (warp == 9) {
        // ---------------- loader: bulk async copies of the operand chunks
        if (lane == 0) {
            const uint32_t bytes = (uint32_t)(GR_CH * 4 * (1 + s) + GR_LBLK + 2 * GR_PBLK);
            uint32_t i = 0;
            for (uint64_t c = c0; c < c1; c++, i++) {
                const uint32_t slot = i % GR_CSTAGES;
                if (i >= GR_CSTAGES) mbar_wait(&S.cempty[slot], ((i / GR_CSTAGES) - 1) & 1);
                GramChunk& C = S.ch[slot];
                uint64_t* bar = &S.cfull[slot];
                mbar_expect_tx(bar, bytes);
                const uint64_t l0 = c * GR_CH;
                const size_t cr = (size_t)(c % a.ch_per_row);
                bulk_g2s(C.z, a.Z + l0, GR_CH * 4, bar);
                if (s) bulk_g2s(C.w, a.GA + l0, GR_CH * 4, bar);
                bulk_g2s(C.lotb, a.LOTb + cr * GR_LBLK, GR_LBLK, bar);
                bulk_g2s(C.lotp[0], a.LOTp[2 * s] + cr * GR_PBLK, GR_PBLK, bar);
                bulk_g2s(C.lotp[1], a.LOTp[2 * s + 1] + cr * GR_PBLK, GR_PBLK, bar);
            }
        }
    } else if (warp == 8) {
        // ---------------- MMA issuer
        uint32_t it = 0;
        for (uint64_t c = c0; c < c1; c++) {
            const bool seg_first = c == c0 || c % a.ch_per_row == 0;
            const bool seg_last = c + 1 == c1 || (c + 1) % a.ch_per_row == 0;
            for (int kk = 0; kk < GR_CH_KS; kk++, it++) {
                const uint32_t st = it % GR_STAGES;
                mbar_wait(&S.full[st], (it / GR_STAGES) & 1);
                tc_fence_after();
                if (lane == 0) {
                    const uint64_t bd = bdesc(S.sB[st]), bd16 = bdesc(S.sB[st] + 512);   // planes 0.., 16..
                    const uint32_t abase = tmem + GR_ASTAGE + st * GR_STAGE_COLS;
                    const uint32_t acc = !(seg_first && kk == 0);
#pragma unroll
                    for (int t = 0; t < 4; t++) mma_i8(tmem + 32 * t, abase + 8 * t, bd, acc);
#pragma unroll
                    for (int t = 4; t < 8; t++) {
                        if (GR_SYM)
                            mma_i8(tmem + GR_ACC_HI + 16 * (t - 4), abase + 8 * t, bd16, acc, GR_IDESC16);
                        else
                            mma_i8(tmem + 32 * t, abase + 8 * t, bd, acc);
                    }
                    // linear cells: one accumulator per parity of the K step (first use: kk = 0 / 1)
                    mma_i8(tmem + GR_ACC_LIN + 32 * (kk & 1), abase + 64, bd, !(seg_first && kk < 2));
                    mma_commit(&S.empty[st]);
                    if (seg_last && kk == GR_CH_KS - 1) mma_commit(&S.accfull);
                }
                __syncwarp();
            }
        }
    } else {
        // ---------------- operand producers + epilogue
        const int q = warp & 3, grp = warp >> 2;
        constexpr int LGRP = GR_SELFGATE ? 1 : 0;   // the warp group that builds the linear-tile rows
        const bool lin = grp == LGRP && q < 3;   // this warp also builds the linear-cell tile rows (q: 0 = E'_x1,
                                              // 1 = E'_x2 o(own entry), 2 = E'_x2 o(pair partner))
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        uint32_t it = 0, seg = 0, ci = 0;
        for (uint64_t c = c0; c < c1; c++, ci++) {
            const uint32_t slot = ci % GR_CSTAGES;
            const uint64_t row = c / a.ch_per_row;
            const bool seg_last = c + 1 == c1 || (c + 1) % a.ch_per_row == 0;
            mbar_wait(&S.cfull[slot], (ci / GR_CSTAGES) & 1);
            const GramChunk& C = S.ch[slot];
            const uint32_t* Wsm = s ? C.w : C.z;
            for (int kk = 0; kk < GR_CH_KS; kk++, it++) {
                const uint32_t st = it % GR_STAGES, par = it & 1;
                // K step kk: entries 64 (kk / 2) + 2 m + (kk & 1), m = lane (the pair 32 (kk / 2) + m of the chunk)
                const uint32_t ei = 64 * (kk >> 1) + 2 * lane + (kk & 1);
                const uint32_t wv = Wsm[ei] & a.qr_mask;
                uint32_t zv = 0, zo = 0;   // sign words of the entries and of their pair partners: the gate warp
                if (!GR_SELFGATE && warp == GR_GATE_WARP) {
                    zv = C.z[ei];
                    zo = C.z[ei ^ 1];
                }
                uint32_t zg = 0;           // GR_SELFGATE: the sign word this lane's linear row is gated by
                if (GR_SELFGATE && lin && q) zg = C.z[q == 1 ? ei : ei ^ 1];
                const uint4* lb = reinterpret_cast<const uint4*>(&C.lotb[lane * GR_LROW + 32 * kk]);
                const uint4 b0 = lb[0], b1 = lb[1];
                uint4 x0 = make_uint4(0, 0, 0, 0), x1 = x0;
                if (lin) {
                    const uint4* lx = reinterpret_cast<const uint4*>(&C.lotp[q ? 1 : 0][lane * GR_PROW + 32 * (kk >> 1)]);
                    x0 = lx[0];
                    x1 = lx[1];
                }
                if (kk == GR_CH_KS - 1) {   // last reads of this chunk are in registers: release the slot
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&S.cempty[slot]);
                }
                // phase 1: bit planes 4w..4w+3 -> masks and the B tile
                uint32_t pl[4];
#pragma unroll
                for (int jj = 0; jj < 4; jj++) pl[jj] = __ballot_sync(0xffffffffu, (wv >> (4 * warp + jj)) & 1u);
                uint32_t sigp = 0, sigo = 0, sg = 0;
                if (GR_SELFGATE && lin && q) sg = __ballot_sync(0xffffffffu, (zg >> a.sig_bit) & 1u);
                if (!GR_SELFGATE && warp == GR_GATE_WARP) {
                    sigp = __ballot_sync(0xffffffffu, (zv >> a.sig_bit) & 1u);
                    sigo = __ballot_sync(0xffffffffu, (zo >> a.sig_bit) & 1u);
                }
                if (it >= GR_STAGES) mbar_wait(&S.empty[st], ((it / GR_STAGES) - 1) & 1);
                {
                    const int jj = lane >> 3, c = lane & 7, j = 4 * warp + jj;
                    const uint32_t P = jj == 0 ? pl[0] : jj == 1 ? pl[1] : jj == 2 ? pl[2] : pl[3];
                    const uint32_t m = expand4((P >> (4 * c)) & 15u);
                    S.mask[par][j][c] = m;
                    *reinterpret_cast<uint32_t*>(&S.sB[st][(j >> 3) * 256 + ((4 * c) >> 4) * 128 + (j & 7) * 16 + ((4 * c) & 15)]) =
                        m & 0x01010101u;
                    if (!GR_SELFGATE && warp == GR_GATE_WARP && lane < 8)
                        S.gate[par][lane] = expand4(((~sigp) >> (4 * lane)) & 15u);
                    if (!GR_SELFGATE && warp == GR_GATE_WARP && lane >= 8 && lane < 16)
                        S.gate2[par][lane - 8] = expand4(((~sigo) >> (4 * (lane - 8))) & 15u);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("bar.sync 1, 256;" ::: "memory");
                // phase 2: A tiles into TMEM
                const uint32_t lo[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                const uint32_t abase = tmem + lane_base + GR_ASTAGE + st * GR_STAGE_COLS;
#pragma unroll
                for (int tt = 0; tt < 4; tt++) {
                    const int t = 4 * grp + tt, j1 = 4 * t + q;
                    const uint4 m0 = *reinterpret_cast<const uint4*>(&S.mask[par][j1][0]);
                    const uint4 m1 = *reinterpret_cast<const uint4*>(&S.mask[par][j1][4]);
                    const uint32_t w8[8] = {lo[0] & m0.x, lo[1] & m0.y, lo[2] & m0.z, lo[3] & m0.w,
                                            lo[4] & m1.x, lo[5] & m1.y, lo[6] & m1.z, lo[7] & m1.w};
                    tmem_st8(abase + 8 * t, w8);
                }
                if (grp == LGRP) {   // linear-cell tile: rows (q, limb k); q = 3 rows are zero
                    uint32_t w8[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
                    if (GR_SELFGATE && (q == 1 || q == 2)) {
#pragma unroll
                        for (int c = 0; c < 8; c++) w8[c] &= expand4(((~sg) >> (4 * c)) & 15u);
                    } else if (q == 1 || q == 2) {
                        const uint32_t* gp = q == 1 ? S.gate[par] : S.gate2[par];
                        const uint4 g0 = *reinterpret_cast<const uint4*>(&gp[0]);
                        const uint4 g1 = *reinterpret_cast<const uint4*>(&gp[4]);
                        w8[0] &= g0.x; w8[1] &= g0.y; w8[2] &= g0.z; w8[3] &= g0.w;
                        w8[4] &= g1.x; w8[5] &= g1.y; w8[6] &= g1.z; w8[7] &= g1.w;
                    }
                    tmem_st8(abase + 64, w8);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.full[st]);
            }
            if (!seg_last) continue;
            // ---- segment epilogue: 32 limb sums per cell -> Fr, times HI[row]
            mbar_wait(&S.accfull, seg & 1);
            seg++;
            tc_fence_after();
            uint32_t (*stg)[33] = S.stage[warp];
            for (int tt = 0; tt < 4; tt++) {
                const int t = 4 * grp + tt, j1 = 4 * t + q;
                if (grp == 0) {   // N = 32 tiles: column j2 = lane
                    uint32_t v[32];
                    tmem_ld32(tmem + lane_base + 32 * t, v);
#pragma unroll
                    for (int c = 0; c < 32; c++) stg[c][lane] = v[c];
                } else {          // N = 16 tiles (j1 >= 16): column j2 = 16 + lane
                    uint32_t v[16];
                    tmem_ld16(tmem + lane_base + (GR_SYM ? GR_ACC_HI + 16 * (t - 4) : 32 * t + 16), v);
#pragma unroll
                    for (int c = 0; c < 16; c++) stg[c][lane] = v[c];
                }
                __syncwarp();
                const int j2 = grp == 0 ? lane : 16 + lane;
                if (j1 < (int)B && j2 >= j1 && j2 < (int)B && (grp == 0 || lane < 16)) {
                    fr_t val = fr_mul(compose_limbs(stg[grp == 0 ? j2 : lane]), fr_load(&a.HI[4][row]));
                    fr_t& dst = S.tot[6 * B + gr_tri(j1, j2, B)];
                    dst = fr_add(dst, val);
                }
                __syncwarp();
            }
            if (grp == LGRP && q < 3) {
                for (int par = 0; par < 2; par++) {
                    uint32_t v[32];
                    tmem_ld32(tmem + lane_base + GR_ACC_LIN + 32 * par, v);
#pragma unroll
                    for (int c = 0; c < 32; c++) stg[c][lane] = v[c];
                    __syncwarp();
                    const int j = lane;
                    if (j < (int)B) {
                        fr_t val = fr_mul(compose_limbs(stg[j]), fr_load(&a.HI[2 * s + (q ? 1 : 0)][row]));
                        fr_t& dst = S.tot[(par * 3 + q) * B + j];
                        dst = fr_add(dst, val);
                    }
                    __syncwarp();
                }
            }
            tc_fence_before();
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    fr_t* out = a.partials + ((size_t)s * a.G + g) * ncs;
    for (uint32_t i = threadIdx.x; i < ncs; i += blockDim.x) fr_store(&out[i], S.tot[i]);
    if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Sums over the G CTAs of a word.  lin6[s][par][q][j] (12 B values, the linear cells per parity) and the Gram
// cells of both words into cell_tot[4B ..) (relu.cu cell_decode order).
// One warp per output: the lanes add strided partials, then a shuffle tree (the 74-long serial chain per thread
// was latency-bound: 41 us).
__global__ void k_relu_gram_reduce(const fr_t* partials, uint32_t G, uint32_t B, fr_t* cell_tot, fr_t* lin6) {
    const uint32_t T = B * (B + 1) / 2, ncs = 6 * B + T, nout = 12 * B + 2 * T;
    const uint32_t lane = threadIdx.x & 31, nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nout; c += nw) {
        uint32_t s, local;
        fr_t* dst;
        if (c < 12 * B) {
            s = c / (6 * B);
            local = c % (6 * B);
            dst = &lin6[c];
        } else {
            s = (c - 12 * B) / T;
            local = 6 * B + (c - 12 * B) % T;
            dst = &cell_tot[4 * B + (c - 12 * B)];
        }
        fr_t acc[1] = {fr_zero()};
        for (uint32_t gg = lane; gg < G; gg += 32) acc[0] = fr_add(acc[0], fr_load(&partials[((size_t)s * G + gg) * ncs + local]));
        warp_reduce_fr<1>(acc);
        if (lane == 0) fr_store(dst, acc[0]);
    }
}

// The j-phase's linear cells M_x[j] = beta(u_x[0], 0) Lin[s][0][q][j] + beta(u_x[0], 1) Lin[s][1][q][j], x = 2 s + q
// (q < 2: the own-entry gate), into cell_tot[0, 4B)
struct GramU0 {
    const fr_t* u[4];
};
__global__ void k_relu_gram_lin(const fr_t* lin6, uint32_t B, GramU0 U, fr_t* cell_tot) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= 4 * B) return;
    const uint32_t x = c / B, j = c % B, s = x >> 1, q = x & 1;
    const fr_t u0 = fr_load(&U.u[x][0]);
    const fr_t e = fr_load(&lin6[(s * 6 + q) * B + j]), o = fr_load(&lin6[(s * 6 + 3 + q) * B + j]);
    fr_store(&cell_tot[c], fr_add(e, fr_mul(u0, fr_sub(o, e))));   // (1 - u0) e + u0 o
}

// e_b's LO table, limb-transposed with the entries of a chunk in K-step order: entry 64 g + 2 m + par of the
// chunk at position 32 (2 g + par) + m:  LOT[(l / 256) * GR_LBLK + k * GR_LROW + pos] = byte k of LO[l]
__global__ void k_lo_limbs_perm(const fr_t* LO, uint32_t n, uint8_t* LOT) {
    for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < n; l += gridDim.x * blockDim.x) {
        const fr_t v = fr_load(&LO[l]);
        const uint32_t e = l % GR_CH, g = e >> 6, r = e & 63;
        const uint32_t pos = 32 * (2 * g + (r & 1)) + (r >> 1);
        uint8_t* dst = LOT + (size_t)(l / GR_CH) * GR_LBLK + pos;
#pragma unroll
        for (int k = 0; k < 32; k++) dst[k * GR_LROW] = (uint8_t)(v.v[k >> 2] >> (8 * (k & 3)));
    }
}
// a pair table (n pairs), limb-transposed in chunks of 128 pairs: LOTp[(l / 128) * GR_PBLK + k * GR_PROW + l % 128]
__global__ void k_lo_limbs_pairs(const fr_t* LO, uint32_t n, uint8_t* LOT) {
    for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < n; l += gridDim.x * blockDim.x) {
        const fr_t v = fr_load(&LO[l]);
        uint8_t* dst = LOT + (size_t)(l / GR_PCH) * GR_PBLK + (l % GR_PCH);
#pragma unroll
        for (int k = 0; k < 32; k++) dst[k * GR_PROW] = (uint8_t)(v.v[k >> 2] >> (8 * (k & 3)));
    }
}

bool relu_gram_supported(uint32_t logD, uint32_t B) { return logD >= 12 && B >= 8 && B <= 32; }

void relu_bitsums_gram(zk_ctx* ctx, const int32_t* Z, const int32_t* GA, uint32_t logD, uint32_t qr_mask,
                       uint32_t sig_bit, uint32_t B, const fr_t* const u_i[5], fr_t* cell_tot, fr_t* lin6, Scratch& s) {
    const uint32_t lo_bits = logD < 16 ? logD : 16, hi_bits = logD - lo_bits;
    const uint32_t lo_n = 1u << lo_bits;
    GramArgs ga;
    memset(&ga, 0, sizeof ga);
    fr_t* los[5];
    EqJob jobs[10];
    for (int x = 0; x < 5; x++) {   // the ten eq tables in two launches: e_b over the segment's lo_bits
        // variables; E'_x (x < 4) over its pairs (variables 1 .. lo_bits - 1; variable 0 is the first i-round's)
        const uint32_t k = x == 4 ? lo_bits : lo_bits - 1;
        los[x] = s.alloc<fr_t>(1ull << k);
        fr_t* hi = s.alloc<fr_t>(1ull << hi_bits);
        jobs[2 * x] = EqJob{u_i[x] + (x == 4 ? 0 : 1), k, nullptr, 1, los[x]};
        jobs[2 * x + 1] = EqJob{u_i[x] + lo_bits, hi_bits, nullptr, 0, hi};
        ga.HI[x] = hi;
    }
    eq_tables_batch(ctx, 10, jobs, s);
    uint8_t* lotb = s.alloc<uint8_t>((size_t)(lo_n / GR_CH) * GR_LBLK);
    ZK_LAUNCH(ctx, k_lo_limbs_perm, grid_for(ctx, lo_n, 256, 4), 256, 0, (const fr_t*)los[4], lo_n, lotb);
    ga.LOTb = lotb;
    for (int x = 0; x < 4; x++) {
        uint8_t* lot = s.alloc<uint8_t>((size_t)(lo_n / GR_CH) * GR_PBLK);
        ZK_LAUNCH(ctx, k_lo_limbs_pairs, grid_for(ctx, lo_n / 2, 256, 4), 256, 0, (const fr_t*)los[x], lo_n / 2, lot);
        ga.LOTp[x] = lot;
    }
    ga.Z = Z;
    ga.GA = GA;
    ga.nch = (1ull << logD) / GR_CH;
    ga.ch_per_row = lo_n / GR_CH;
    ga.qr_mask = qr_mask;
    ga.sig_bit = sig_bit;
    ga.B = B;
    // CTAs per word: G = num_sms / 2 x ZKDL_GRAM_WAVES (one CTA per SM; more waves = finer work, less exposed to
    // SMs held by other streams' kernels)
    static const int waves = getenv("ZKDL_GRAM_WAVES") ? atoi(getenv("ZKDL_GRAM_WAVES")) : 1;
    uint32_t G = (uint32_t)ctx->num_sms / 2 * (uint32_t)(waves < 1 ? 1 : waves);
    if ((uint64_t)G > ga.nch) G = (uint32_t)ga.nch;
    ga.G = G;
    const uint32_t T = B * (B + 1) / 2, ncs = 6 * B + T;
    ga.partials = s.alloc<fr_t>(2ull * G * ncs);
    // > half the SM's shared memory: one CTA per SM, so the 512-column TMEM allocation never waits
    const size_t smem = sizeof(GramSmem) + 1024 > 120 * 1024 ? sizeof(GramSmem) + 1024 : 120 * 1024;
    ZK_CUDA(cudaFuncSetAttribute(k_relu_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ZK_LAUNCH(ctx, k_relu_gram, 2 * G, 320, smem, ga);
    ZK_LAUNCH(ctx, k_relu_gram_reduce, (12 * B + 2 * T + 7) / 8, 256, 0, (const fr_t*)ga.partials, G, B, cell_tot, lin6);
    GramU0 U;
    for (int x = 0; x < 4; x++) U.u[x] = u_i[x];
    ZK_LAUNCH(ctx, k_relu_gram_lin, (4 * B + 127) / 128, 128, 0, (const fr_t*)lin6, B, U, cell_tot);
}

}  // namespace zk
