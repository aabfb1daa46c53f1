// relu.cu — zkReLU on the B200 (PAPER §3, App. A).
//
// Statement (D3b, D5, D10, D13): variables x = (j, i), j = bit position (logB bits, bound first),
// i = entry (logD bits):
//   sum_{i,j} [ r^2 E_Z(i) a0 s(j) + r E_A(i) (1-sig(i)) a0 s'(j) + E_b(i,j)(a0^2 - a0)
//             + r'r^2 E_GA(i) a1 s(j) + r'r E_GZ(i) (1-sig(i)) a1 s'(j) + r' E_b(i,j)(a1^2 - a1) ]
//   = r^2 Z~(u_Z) + r A~(u_A) + r'r^2 G_A~(u_GA) + r'r G_Z~(u_GZ)
// with a0(i,j) = bit j of Z_i, a1(i,j) = bit j of G_A_i (two's complement, Q+R bits), sig = bit Q+R-1
// of Z, E_x(i) = beta(u_x, i), E_b(i,j) = beta(u_bin, (j, i)).
//
// Prover algorithm ("bits first"; the transcript is the statement's unique one, D18):
//  * j-rounds: every j-round polynomial is a function of four linear sums M_x[j] = sum_i c_x(i) bit_j
//    and two 32x32 co-occurrence matrices C_s[j1][j2] = sum_i e_b(i) bit_j1 bit_j2 (L_s = diag C_s),
//    because a0~(i, rho)^2 = sum_{j1,j2} beta(rho,j1) beta(rho,j2) bit_j1 bit_j2 and
//    E_b(i, j) = beta(u_bin_j, j) beta(u_bin_i, i).  One pass over the int32 words computes them with
//    masked lazy additions (no Fr multiplication per entry); the 5 rounds then run on 32-entry
//    vectors and a 32x32 matrix in one CTA (bilinear fold for C).
//  * i-rounds: after the j-rounds, a0(i) = sum_j beta(r_j, j) bit_j(Z_i) = sum of 4 byte-table lookups;
//    the remaining logD rounds are a degree-3 sumcheck over a0, a1, 1-sig and five eq tables held as
//    LO (low variables, pair-summed in the round kernel) x HI (<= 5 variables, rescaled by
//    beta(u_t, r_t) in the finalizer), so no 2^logD eq table is ever written.
#include "relu.cuh"
#include "tables.cuh"

namespace zk {

// ---------------------------------------------------------------- row a7: tables
__global__ void k_relu_tables(const int32_t* Z, const int32_t* GA, uint64_t D, uint32_t Q, uint32_t R, uint8_t* sign,
                              int32_t* A, int32_t* GZ, int32_t* Zp, int32_t* GAp, int32_t* RZ, int32_t* RGA,
                              unsigned int* bad) {
    const int64_t lim = 1ll << (Q + R - 1);
    const int64_t half = 1ll << (R - 1);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < D; i += (uint64_t)gridDim.x * blockDim.x) {
        int64_t z = Z[i], g = GA[i];
        if (z < -lim || z >= lim || g < -lim || g >= lim) atomicOr(bad, 1u);
        int64_t zp = (z + half) >> R, gp = (g + half) >> R;   // half-up rounding (D9)
        bool neg = z < 0;                                      // sign of Z gates both (D10)
        sign[i] = neg;
        A[i] = neg ? 0 : (int32_t)zp;
        GZ[i] = neg ? 0 : (int32_t)gp;
        if (Zp) Zp[i] = (int32_t)zp;
        if (GAp) GAp[i] = (int32_t)gp;
        if (RZ) RZ[i] = (int32_t)(z - (zp << R));
        if (RGA) RGA[i] = (int32_t)(g - (gp << R));
    }
}

bool relu_tables_dev(zk_ctx* ctx, const int32_t* Z, const int32_t* GA, uint64_t D, uint32_t Q, uint32_t R, uint8_t* sign,
                     int32_t* A, int32_t* GZ, int32_t* Zp, int32_t* GAp, int32_t* RZ, int32_t* RGA, Scratch& s) {
    unsigned int* bad = s.alloc_zero<unsigned int>(1);
    if (D) ZK_LAUNCH(ctx, k_relu_tables, grid_for(ctx, D, 256, 8), 256, 0, Z, GA, D, Q, R, sign, A, GZ, Zp, GAp, RZ, RGA, bad);
    unsigned int h = 0;
    ZK_CUDA(cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, ctx->stream));
    ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    return h == 0;
}

__global__ void k_relu_range(const int32_t* Z, const int32_t* GA, uint64_t D, uint32_t QR, unsigned int* bad) {
    const int64_t lim = 1ll << (QR - 1);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < D; i += (uint64_t)gridDim.x * blockDim.x) {
        int64_t z = Z[i], g = GA[i];
        if (z < -lim || z >= lim || g < -lim || g >= lim) atomicOr(bad, 1u);
    }
}

// ---------------------------------------------------------------- bit sums for the j-rounds
// A cell accumulates sum_i c_lot(i) [ (word_i & m1) == m1 ] [ !(gate && sig_i) ].
struct BitCell {
    uint32_t m1;
    uint8_t word;   // 0: Z, 1: G_A
    uint8_t gate;   // multiply by (1 - sig)
    uint8_t lot;    // eq table: 0 Z, 1 A, 2 GA, 3 GZ, 4 b
    uint8_t pad;
};

struct BitsumArgs {
    const int32_t* Z;
    const int32_t* GA;
    uint32_t logD, lo_bits, qr_mask, sig_bit;
    const fr_t* LO[5];   // eq over the low lo_bits variables, scaled by R (lazy accumulation)
    const fr_t* HI[5];   // eq over the remaining variables
    uint32_t B, ncell;   // cells decoded from their index (cell_decode)
    fr_t* partials;      // gridDim.x * ncell
};

// Cell c of the bit-sum list: [0, 4B) linear cells M_x[j] (x = c / B: 0 Z, 1 A, 2 G_A, 3 G_Z; word Z
// for x < 2, G_A otherwise), then the co-occurrence cells C_s[j1][j2] (j1 <= j2, row-major upper
// triangles, s = 0 then 1) -- the same order k_relu_jrounds reads (tri_index).
__device__ __forceinline__ void cell_decode(uint32_t c, uint32_t B, uint32_t& j1, uint32_t& j2, uint32_t& s,
                                            uint32_t& x) {
    if (c < 4 * B) {
        x = c / B;
        j1 = j2 = c % B;
        s = x >= 2;
        return;
    }
    uint32_t idx = c - 4 * B;
    const uint32_t T = B * (B + 1) / 2;
    s = idx / T;
    idx -= s * T;
    x = 4;
    uint32_t j = 0;
    while (idx >= B - j) {
        idx -= B - j;
        j++;
    }
    j1 = j;
    j2 = j + idx;
}

__device__ __forceinline__ BitCell bitcell_at(uint32_t c, uint32_t B, uint32_t QR) {
    uint32_t j1, j2, s, x;
    cell_decode(c, B, j1, j2, s, x);
    BitCell r;
    r.m1 = (j1 < QR && j2 < QR) ? ((1u << j1) | (1u << j2)) : 0xffffffffu;   // padding columns never match
    r.word = (uint8_t)s;
    r.gate = (uint8_t)(x == 1 || x == 3);
    r.lot = (uint8_t)x;
    r.pad = 0;
    return r;
}

constexpr int BS_CH = 128;   // entries staged per chunk

__device__ __forceinline__ void masked_add10(uint32_t (&a)[10], const fr_t& v, uint32_t mm) {
    asm("add.cc.u32  %0, %0, %10;\n\t"
        "addc.cc.u32 %1, %1, %11;\n\t"
        "addc.cc.u32 %2, %2, %12;\n\t"
        "addc.cc.u32 %3, %3, %13;\n\t"
        "addc.cc.u32 %4, %4, %14;\n\t"
        "addc.cc.u32 %5, %5, %15;\n\t"
        "addc.cc.u32 %6, %6, %16;\n\t"
        "addc.cc.u32 %7, %7, %17;\n\t"
        "addc.cc.u32 %8, %8, 0;\n\t"
        "addc.u32    %9, %9, 0;"
        : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
          "+r"(a[8]), "+r"(a[9])
        : "r"(v.v[0] & mm), "r"(v.v[1] & mm), "r"(v.v[2] & mm), "r"(v.v[3] & mm), "r"(v.v[4] & mm),
          "r"(v.v[5] & mm), "r"(v.v[6] & mm), "r"(v.v[7] & mm));
}

// ---------------------------------------------------------------- bit sums, subset-sum tables (v2)
// Per chunk of 64 entries (within one LO row): byte planes P[s][g][j] (bit j of the 8 words of
// byte-group g), byte subset-sum tables Tb[g][v] = sum_{k in v} e_b(8g + k) for the co-occurrence
// cells, nibble tables Tm[x][h][v] = sum_{k in v} c_x(4h + k) for the linear cells.  A C cell
// (j1, j2) then costs one lookup Tb[g][P[g][j1] & P[g][j2]] and one lazy 320-bit add per 8 entries,
// an M cell one lookup per 4 entries; the tables cost ~2.5 Fr additions per entry for all cells.
// Table entries are sums of LO' values (eq * R, "double Montgomery"), reduced mod p; the lazy
// accumulators are closed with REDC (-> Montgomery) and multiplied by HI[row] when the row changes.
constexpr int BS2_CH = 64;
constexpr int BS2_T = 512;
constexpr int BS2_MAXC = 3;   // cell slots per thread: cells tid, tid + 512, tid + 1024

struct BitCell2 {
    uint8_t j1, j2, s, x;   // bit positions, word (0 Z, 1 G_A), weight table (M cells: 0..3; C cells: 4)
};

struct Bitsum2Args {
    const int32_t* Z;
    const int32_t* GA;
    uint32_t logD, lo_bits, qr_mask, sig_bit;
    const fr_t* LO[5];
    const fr_t* HI[5];
    uint32_t B;              // cells decoded from their index: [0, nM) linear, [nM, nM + nC) co-occurrence
    uint32_t nM, nC;
    fr_t* partials;          // gridDim.x * (nM + nC), zero-initialised; per-block running totals
};

struct Bitsum2Smem {
    fr_t Tb[8][256];
    fr_t Tm[4][16][16];
    fr_t E[5][BS2_CH];
    fr_t U[8][8];
    uint64_t P64[2][32];     // [s][j]: byte g = bit j of the 8 words of group g
    uint32_t W[2][BS2_CH];
    uint8_t sig[BS2_CH];
};

__device__ __forceinline__ void wide_add_fr(uint32_t (&a)[10], const fr_t& v) {
    asm("add.cc.u32  %0, %0, %10;\n\t"
        "addc.cc.u32 %1, %1, %11;\n\t"
        "addc.cc.u32 %2, %2, %12;\n\t"
        "addc.cc.u32 %3, %3, %13;\n\t"
        "addc.cc.u32 %4, %4, %14;\n\t"
        "addc.cc.u32 %5, %5, %15;\n\t"
        "addc.cc.u32 %6, %6, %16;\n\t"
        "addc.cc.u32 %7, %7, %17;\n\t"
        "addc.cc.u32 %8, %8, 0;\n\t"
        "addc.u32    %9, %9, 0;"
        : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
          "+r"(a[8]), "+r"(a[9])
        : "r"(v.v[0]), "r"(v.v[1]), "r"(v.v[2]), "r"(v.v[3]), "r"(v.v[4]), "r"(v.v[5]), "r"(v.v[6]), "r"(v.v[7]));
}

__device__ __forceinline__ void bs2_flush(uint32_t (&acc)[10], const fr_t* hi, uint64_t row, fr_t* tot) {
    fr_t v = fr_mul(fr_redc_wide(acc), fr_load(&hi[row]));
    fr_store(tot, fr_add(fr_load(tot), v));
#pragma unroll
    for (int k = 0; k < 10; k++) acc[k] = 0;
}

__global__ void __launch_bounds__(BS2_T, 1) k_relu_bitsums2(Bitsum2Args a) {
    extern __shared__ __align__(16) uint8_t smem2_raw[];
    Bitsum2Smem& S = *reinterpret_cast<Bitsum2Smem*>(smem2_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t D = 1ull << a.logD;
    const uint64_t nchunks = D / BS2_CH;
    const uint64_t c_begin = blockIdx.x * nchunks / gridDim.x, c_end = (blockIdx.x + 1) * nchunks / gridDim.x;
    const uint32_t ncell = a.nM + a.nC;
    BitCell2 cl[BS2_MAXC];
    int cid[BS2_MAXC];
#pragma unroll
    for (int q = 0; q < BS2_MAXC; q++) {
        const int c = tid + q * BS2_T;
        cid[q] = c < (int)ncell ? c : -1;
        uint32_t j1 = 0, j2 = 0, s = 0, x = 0;
        if (c < (int)ncell) cell_decode((uint32_t)c, a.B, j1, j2, s, x);
        cl[q] = BitCell2{(uint8_t)j1, (uint8_t)j2, (uint8_t)s, (uint8_t)x};
    }
    fr_t* tot = a.partials + (uint64_t)blockIdx.x * ncell;
    uint32_t acc[BS2_MAXC][10];
#pragma unroll
    for (int q = 0; q < BS2_MAXC; q++)
#pragma unroll
        for (int k = 0; k < 10; k++) acc[q][k] = 0;
    const uint64_t lo_mask = (1ull << a.lo_bits) - 1;
    uint64_t row = (c_begin * BS2_CH) >> a.lo_bits;
    for (uint64_t ch = c_begin; ch < c_end; ch++) {
        const uint64_t i0 = ch * BS2_CH;
        const uint64_t r_here = i0 >> a.lo_bits;
        if (r_here != row) {
#pragma unroll
            for (int q = 0; q < BS2_MAXC; q++)
                if (cid[q] >= 0) bs2_flush(acc[q], a.HI[cl[q].x], row, &tot[cid[q]]);
            row = r_here;
        }
        __syncthreads();
        // stage the chunk: LO' weights, words, sign bits
        if (tid < 5 * BS2_CH) {
            const int x = tid / BS2_CH, k = tid % BS2_CH;
            S.E[x][k] = fr_load(&a.LO[x][(i0 + k) & lo_mask]);
        } else if (tid >= 384 && tid < 384 + BS2_CH) {
            const int k = tid - 384;
            uint32_t z = (uint32_t)__ldg(a.Z + i0 + k), g = (uint32_t)__ldg(a.GA + i0 + k);
            S.W[0][k] = z & a.qr_mask;
            S.W[1][k] = g & a.qr_mask;
            S.sig[k] = (z >> a.sig_bit) & 1;
        }
        __syncthreads();
        // gate c_A, c_GZ by (1 - sig); bit planes; U
        if (tid < 2 * BS2_CH) {
            const int k = tid % BS2_CH, x = tid < BS2_CH ? 1 : 3;
            if (S.sig[k]) S.E[x][k] = fr_zero();
        } else if (tid >= 128 && tid < 192) {
            const int e = tid - 128, sd = e >> 5, j = e & 31;
            uint64_t m = 0;
#pragma unroll
            for (int k = 0; k < BS2_CH; k++) m |= (uint64_t)((S.W[sd][k] >> j) & 1u) << k;
            S.P64[sd][j] = m;   // bit k of the chunk = byte k/8, bit k%8: byte g holds group g
        } else if (tid >= 256 && tid < 256 + 64) {
            const int g = (tid - 256) >> 3, q = (tid - 256) & 7;
            const fr_t* eb = &S.E[4][8 * g + 5];
            fr_t u = fr_zero();
            if (q & 1) u = eb[0];
            if (q & 2) u = fr_add(u, eb[1]);
            if (q & 4) u = fr_add(u, eb[2]);
            S.U[g][q] = u;
        }
        __syncthreads();
        if (warp < 8) {   // byte tables: warp g builds Tb[g][l + 32 q] = base(l) + U[g][q]
            const int g = warp;
            const fr_t* eb = &S.E[4][8 * g];
            fr_t base = fr_zero();
#pragma unroll
            for (int k = 0; k < 5; k++)
                if ((lane >> k) & 1) base = fr_add(base, eb[k]);
            S.Tb[g][lane] = base;
#pragma unroll
            for (int q = 1; q < 8; q++) S.Tb[g][lane + 32 * q] = fr_add(base, S.U[g][q]);
        } else {          // nibble tables Tm[x][h][v]
            for (int e = tid - 256; e < 4 * 16 * 16; e += 256) {
                const int x = e >> 8, h = (e >> 4) & 15, v = e & 15;
                const fr_t* cx = &S.E[x][4 * h];
                fr_t t = fr_zero();
#pragma unroll
                for (int k = 0; k < 4; k++)
                    if ((v >> k) & 1) t = fr_add(t, cx[k]);
                S.Tm[x][h][v] = t;
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < BS2_MAXC; q++) {
            if (cid[q] < 0) continue;
            if (cid[q] < (int)a.nM) {   // linear cell: 16 nibble lookups
                const uint64_t pm = S.P64[cl[q].s][cl[q].j1];
                const int x = cl[q].x;
#pragma unroll 4
                for (int h = 0; h < 16; h++) wide_add_fr(acc[q], S.Tm[x][h][(pm >> (4 * h)) & 15]);
            } else {                     // co-occurrence cell: 8 byte lookups
                const uint64_t pm = S.P64[cl[q].s][cl[q].j1] & S.P64[cl[q].s][cl[q].j2];
#pragma unroll
                for (int g = 0; g < 8; g++) wide_add_fr(acc[q], S.Tb[g][(pm >> (8 * g)) & 255]);
            }
        }
    }
    if (c_begin < c_end) {
#pragma unroll
        for (int q = 0; q < BS2_MAXC; q++)
            if (cid[q] >= 0) bs2_flush(acc[q], a.HI[cl[q].x], row, &tot[cid[q]]);
    }
}

// Each thread owns cells tid and tid + blockDim.x.  Each block walks a contiguous range of chunks;
// the lazy accumulators are closed (REDC, times HI[row]) whenever the row i >> lo_bits changes.
__global__ void __launch_bounds__(640) k_relu_bitsums(BitsumArgs a) {
    extern __shared__ uint8_t smem_raw[];
    fr_t* sLO = reinterpret_cast<fr_t*>(smem_raw);                       // [5][BS_CH]
    uint32_t* sW = reinterpret_cast<uint32_t*>(sLO + 5 * BS_CH);          // [2][BS_CH]
    uint8_t* sSig = reinterpret_cast<uint8_t*>(sW + 2 * BS_CH);           // [BS_CH]
    const uint64_t D = 1ull << a.logD;
    const uint64_t CH = D < BS_CH ? D : BS_CH;
    const uint64_t nchunks = D / CH;
    const uint64_t c_begin = blockIdx.x * nchunks / gridDim.x, c_end = (blockIdx.x + 1) * nchunks / gridDim.x;
    BitCell cell[2];
    bool have[2];
    for (int q = 0; q < 2; q++) {
        uint32_t c = threadIdx.x + q * blockDim.x;
        have[q] = c < a.ncell;
        cell[q] = have[q] ? bitcell_at(c, a.B, a.sig_bit + 1) : BitCell{0, 0, 0, 0, 0};
    }
    uint32_t acc[2][10];
    fr_t tot[2] = {fr_zero(), fr_zero()};
    for (int q = 0; q < 2; q++)
        for (int k = 0; k < 10; k++) acc[q][k] = 0;
    const uint64_t lo_mask = (1ull << a.lo_bits) - 1;
    uint64_t row = c_begin * CH >> a.lo_bits;
    for (uint64_t ch = c_begin; ch < c_end; ch++) {
        const uint64_t i0 = ch * CH;
        const uint64_t r_here = i0 >> a.lo_bits;
        if (r_here != row) {
            for (int q = 0; q < 2; q++)
                if (have[q]) {
                    tot[q] = fr_add(tot[q], fr_mul(fr_redc_wide(acc[q]), fr_load(&a.HI[cell[q].lot][row])));
                    for (int k = 0; k < 10; k++) acc[q][k] = 0;
                }
            row = r_here;
        }
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < 5 * CH; e += blockDim.x) {
            uint32_t lot = e / CH, k = e % CH;
            fr_store(&sLO[lot * BS_CH + k], fr_load(&a.LO[lot][(i0 + k) & lo_mask]));
        }
        for (uint32_t k = threadIdx.x; k < CH; k += blockDim.x) {
            uint32_t z = (uint32_t)__ldg(a.Z + i0 + k), g = (uint32_t)__ldg(a.GA + i0 + k);
            sW[k] = z & a.qr_mask;
            sW[BS_CH + k] = g & a.qr_mask;
            sSig[k] = (z >> a.sig_bit) & 1;
        }
        __syncthreads();
        for (uint32_t k = 0; k < CH; k++) {
            const uint32_t sg = sSig[k];
#pragma unroll
            for (int q = 0; q < 2; q++) {
                const uint32_t w = sW[cell[q].word * BS_CH + k];
                const bool on = have[q] && ((w & cell[q].m1) == cell[q].m1) && !(cell[q].gate && sg);
                const fr_t v = sLO[cell[q].lot * BS_CH + k];
                masked_add10(acc[q], v, on ? 0xffffffffu : 0u);
            }
        }
    }
    if (c_begin < c_end)
        for (int q = 0; q < 2; q++)
            if (have[q]) tot[q] = fr_add(tot[q], fr_mul(fr_redc_wide(acc[q]), fr_load(&a.HI[cell[q].lot][row])));
    for (int q = 0; q < 2; q++)
        if (have[q]) fr_store(&a.partials[(uint64_t)blockIdx.x * a.ncell + threadIdx.x + q * blockDim.x], tot[q]);
}

__global__ void k_relu_bitsums_reduce(const fr_t* partials, uint32_t nblocks, uint32_t ncell, fr_t* out) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += gridDim.x * blockDim.x) {
        fr_t s = fr_zero();
        for (uint32_t b = 0; b < nblocks; b++) s = fr_add(s, fr_load(&partials[(uint64_t)b * ncell + c]));
        fr_store(&out[c], s);
    }
}

// ---------------------------------------------------------------- j-rounds (one CTA)
struct JRoundArgs {
    const fr_t* cells;     // cell totals: [0,B) MZ, [B,2B) MA, [2B,3B) MGA, [3B,4B) MGZ, then C0, C1 upper triangles
    uint32_t B, logB, Q, R;
    const fr_t* r;         // r, r'
    const fr_t* ubin;      // u_bin (first logB entries: j variables)
    uint8_t* st;
    uint8_t* msg_out;      // logB rounds x 4 x 32 bytes
    uint8_t* point_out;    // logB x 32 canonical
    fr_t* rj_out;          // logB challenges (Montgomery)
    fr_t* byte_tab;        // ceil(B/8) x 256 entries
    fr_t* kappa;           // [0] kZ [1] kA [2] kGA [3] kGZ [4] kb [5] r' [6] claim after the j-phase
    fr_t* sigma;           // (nullable) the five per-term sums entering the i-phase (Z, A, GA, GZ, b)
    const fr_t* r0cells;   // (nullable, with sigma) lin6 of relu_bitsums_gram: [s][par][q][j]
    fr_t* r0ext;           // the first i-round's linear totals from r0cells (6: Z, A(0), A(inf), GA, GZ(0), GZ(inf))
};

__device__ __forceinline__ int tri_index(int j1, int j2, int B) {   // j1 <= j2, row-major upper triangle
    return j1 * B - j1 * (j1 - 1) / 2 + (j2 - j1);
}

__device__ fr_t small_pow2(int e) {   // Montgomery form of 2^e, 0 <= e < 64
    fr_t b = fr_zero();
    if (e < 32) b.v[0] = 1u << e; else b.v[1] = 1u << (e - 32);
    return fr_mul_cold(ZK_R2, b);
}

__global__ void __launch_bounds__(256) k_relu_jrounds(JRoundArgs a) {
    __shared__ fr_t S[32], SP[32], EB[32], LS[32], LSP[32], LQ[32];
    __shared__ fr_t CQ[32][32];
    __shared__ fr_t vals[64];
    __shared__ fr_t msg[4];
    __shared__ fr_t rt_sm;
    __shared__ fr_t ej[32];
    const int B = a.B, tid = threadIdx.x;
    const int QR = a.Q + a.R;
    const fr_t r = fr_load(&a.r[0]), rp = fr_load(&a.r[1]);
    const fr_t r2 = fr_mul_cold(r, r);
    const fr_t* MZ = a.cells;
    const fr_t* MA = a.cells + B;
    const fr_t* MGA = a.cells + 2 * B;
    const fr_t* MGZ = a.cells + 3 * B;
    const fr_t* C0 = a.cells + 4 * B;
    const fr_t* C1 = C0 + B * (B + 1) / 2;
    // initial vectors
    for (int j = tid; j < B; j += blockDim.x) {
        // s_{Q+R} and s', zero-padded to B columns (D12)
        fr_t s = fr_zero(), sp = fr_zero();
        if (j < QR - 1) s = small_pow2(j);
        else if (j == QR - 1) s = fr_neg(small_pow2(QR - 1));
        if (j == (int)a.R - 1) sp = fr_one();
        else if (j >= (int)a.R && j < QR - 1) sp = small_pow2(j - a.R);
        else if (j == QR - 1) sp = fr_neg(small_pow2(a.Q - 1));
        S[j] = s;
        SP[j] = sp;
        fr_t e = fr_one();
        for (uint32_t t = 0; t < a.logB; t++) {
            fr_t u = fr_load(&a.ubin[t]);
            e = fr_mul_cold(e, ((j >> t) & 1) ? u : fr_sub(fr_one(), u));
        }
        EB[j] = e;
        LS[j] = fr_add(fr_mul_cold(r2, fr_load(&MZ[j])), fr_mul_cold(fr_mul_cold(rp, r2), fr_load(&MGA[j])));
        LSP[j] = fr_add(fr_mul_cold(r, fr_load(&MA[j])), fr_mul_cold(fr_mul_cold(rp, r), fr_load(&MGZ[j])));
    }
    for (int e = tid; e < B * B; e += blockDim.x) {
        int j1 = e / B, j2 = e % B;
        int lo = j1 < j2 ? j1 : j2, hi = j1 < j2 ? j2 : j1;
        int ti = tri_index(lo, hi, B);
        fr_t c = fr_add(fr_load(&C0[ti]), fr_mul_cold(rp, fr_load(&C1[ti])));
        CQ[j1][j2] = c;
        if (j1 == j2) LQ[j1] = c;   // L_s = diag(C_s) since bit^2 = bit
    }
    __shared__ FsScratch fs;
    if (tid < 32) fs_begin(fs, a.st);
    __syncthreads();
    __shared__ fr_t claim_sm;   // g_{logB-1}(r_{logB-1}): the claim entering the i-phase
    for (uint32_t t = 0; t < a.logB; t++) {
        const int n = B >> t, np = n >> 1;
        // evaluations: item (b, X)
        if (tid < 4 * np) {   // independent products in three-product out-of-line bodies (latency: this
                              // single-CTA kernel is on the zkReLU family's critical path)
            const int b = tid >> 2, X = tid & 3;
            const fr_t x = fr_from_u32((uint32_t)X), omx = fr_sub(fr_one(), x);
#define DIF(v) fr_sub(v[2 * b + 1], v[2 * b])
            const fr3_t l1 = fr_mul3_ni(x, DIF(S), x, DIF(SP), x, DIF(EB));
            const fr3_t l2 = fr_mul3_ni(x, DIF(LS), x, DIF(LSP), x, DIF(LQ));
#undef DIF
            const fr_t sv = fr_add(S[2 * b], l1.x), spv = fr_add(SP[2 * b], l1.y), ebv = fr_add(EB[2 * b], l1.z);
            const fr_t lsv = fr_add(LS[2 * b], l2.x), lspv = fr_add(LSP[2 * b], l2.y), lqv = fr_add(LQ[2 * b], l2.z);
            // bilinear: sum_{x1,x2} l(x1) l(x2) CQ[2b+x1][2b+x2]
            fr_t c00 = CQ[2 * b][2 * b], c01 = CQ[2 * b][2 * b + 1], c10 = CQ[2 * b + 1][2 * b], c11 = CQ[2 * b + 1][2 * b + 1];
            const fr3_t w = fr_mul3_ni(omx, omx, omx, x, x, x);
            const fr3_t q = fr_mul3_ni(w.x, c00, w.y, fr_add(c01, c10), w.z, c11);
            const fr_t cq = fr_add(q.x, fr_add(q.y, q.z));
            const fr3_t t3 = fr_mul3_ni(sv, lsv, spv, lspv, ebv, fr_sub(cq, lqv));
            vals[tid] = fr_add(fr_add(t3.x, t3.y), t3.z);
        }
        __syncthreads();
        if (tid < 4) {
            fr_t sum = fr_zero();
            for (int b = 0; b < np; b++) sum = fr_add(sum, vals[4 * b + tid]);
            msg[tid] = sum;
        }
        __syncthreads();
        if (tid < 32) {
            fs_absorb_frs(fs, "relu/msg", tid < 4 ? msg[tid & 3] : fr_zero(), 4, a.msg_out + 128ull * t);
            fr_t rt = fs_challenge(fs, "relu/x");
            if (tid == 0) {
                fr_canon_to_bytes(fs.rc, a.point_out + 32ull * t);
                fr_store(&a.rj_out[t], rt);
                rt_sm = rt;
                if (t + 1 == a.logB) {
                    fr_t ev[4] = {msg[0], msg[1], msg[2], msg[3]};
                    claim_sm = interp_small(ev, 3, rt);
                }
            }
        }
        __syncthreads();
        const fr_t rt = rt_sm;
        // fold vectors
        fr_t nv[6];
        if (tid < np) {
            const int b = tid;
#define DIF(v) fr_sub(v[2 * b + 1], v[2 * b])
            const fr3_t f1 = fr_mul3_ni(rt, DIF(S), rt, DIF(SP), rt, DIF(EB));
            const fr3_t f2 = fr_mul3_ni(rt, DIF(LS), rt, DIF(LSP), rt, DIF(LQ));
#undef DIF
            nv[0] = fr_add(S[2 * b], f1.x); nv[1] = fr_add(SP[2 * b], f1.y); nv[2] = fr_add(EB[2 * b], f1.z);
            nv[3] = fr_add(LS[2 * b], f2.x); nv[4] = fr_add(LSP[2 * b], f2.y); nv[5] = fr_add(LQ[2 * b], f2.z);
        }
        // fold CQ: columns then rows, staged through registers (n * np <= 512 = 2 per thread)
        fr_t cv[2];
        int cc = 0;
        for (int e = tid; e < n * np; e += blockDim.x) {
            int i = e / np, c = e % np;
            cv[cc++] = fr_add(CQ[i][2 * c], fr_mul_ni(rt, fr_sub(CQ[i][2 * c + 1], CQ[i][2 * c])));
        }
        __syncthreads();
        cc = 0;
        for (int e = tid; e < n * np; e += blockDim.x) CQ[e / np][e % np] = cv[cc++];
        if (tid < np) {
            S[tid] = nv[0]; SP[tid] = nv[1]; EB[tid] = nv[2]; LS[tid] = nv[3]; LSP[tid] = nv[4]; LQ[tid] = nv[5];
        }
        __syncthreads();
        fr_t rv = fr_zero();
        if (tid < np * np) {
            int b = tid / np, c = tid % np;
            rv = fr_add(CQ[2 * b][c], fr_mul_ni(rt, fr_sub(CQ[2 * b + 1][c], CQ[2 * b][c])));
        }
        __syncthreads();
        if (tid < np * np) CQ[tid / np][tid % np] = rv;
        __syncthreads();
    }
    if (tid < 32) fs_end(fs, a.st);
    if (tid == 0) {
        const fr_t s = S[0], sp = SP[0];
        fr_store(&a.kappa[0], fr_mul_cold(r2, s));
        fr_store(&a.kappa[1], fr_mul_cold(r, sp));
        fr_store(&a.kappa[2], fr_mul_cold(fr_mul_cold(rp, r2), s));
        fr_store(&a.kappa[3], fr_mul_cold(fr_mul_cold(rp, r), sp));
        fr_store(&a.kappa[4], EB[0]);
        fr_store(&a.kappa[5], rp);
        fr_store(&a.kappa[6], claim_sm);
        fr_store(&a.kappa[7], fr_mul_cold(rp, EB[0]));
    }
    // byte tables: T[b][v] = sum_{k<8} [bit k of v] beta(r_j, 8b + k)
    for (int j = tid; j < B; j += blockDim.x) {
        fr_t e = fr_one();
        for (uint32_t t = 0; t < a.logB; t++) {
            fr_t u = fr_load(&a.rj_out[t]);
            e = fr_mul_cold(e, ((j >> t) & 1) ? u : fr_sub(fr_one(), u));
        }
        ej[j] = e;
    }
    __syncthreads();
    if (a.sigma) {
        // per-term sums entering the i-phase (the derived-X=1 i-rounds): with e_j = beta(r_j, j),
        //   sigma_x = kappa_x sum_j e_j M_x[j]                       (x = Z, A, GA, GZ: the linear cells)
        //   sigma_b = kappa_b (S_0 - L_0) + kappa_b' (S_1 - L_1),     S_s = sum_{j1,j2} e_j1 e_j2 C_s[j1][j2],
        //                                                            L_s = sum_j e_j C_s[j][j]
        // (sum_i e_b(i) a(i)(a(i) - 1) through the Gram cells; their total is the claim kappa[6])
        fr_t (*linp)[32] = CQ;   // (the j-rounds are done with CQ: rows 0-3 hold the linear products)
        if (tid < 4 * B) {
            const int x = tid / B, j = tid % B;
            linp[x][j] = fr_mul_ni(ej[j], fr_load(&a.cells[x * B + j]));
        }
        fr_t gacc[2] = {fr_zero(), fr_zero()};
        const int T = B * (B + 1) / 2;
        for (int e = tid; e < T; e += blockDim.x) {
            int j1 = 0, rem = e;
            while (rem >= B - j1) {
                rem -= B - j1;
                j1++;
            }
            const int j2 = j1 + rem;
            fr_t w = fr_mul_ni(ej[j1], ej[j2]);
            w = j1 == j2 ? fr_sub(w, ej[j1]) : fr_add(w, w);
            const fr2p_t c = fr_mul2_ni(w, fr_load(&C0[e]), w, fr_load(&C1[e]));
            gacc[0] = fr_add(gacc[0], c.x);
            gacc[1] = fr_add(gacc[1], c.y);
        }
        block_reduce_fr<2>(gacc, vals);   // (vals: 64 elements, free after the j-rounds)
        if (tid < 4) {
            fr_t acc = fr_zero();
            for (int j = 0; j < B; j++) acc = fr_add(acc, linp[tid][j]);
            const fr_t s = S[0], sp = SP[0];
            const fr_t k = tid == 0 ? fr_mul_ni(r2, s) : tid == 1 ? fr_mul_ni(r, sp) :
                           tid == 2 ? fr_mul_ni(fr_mul_ni(rp, r2), s) : fr_mul_ni(fr_mul_ni(rp, r), sp);
            fr_store(&a.sigma[tid], fr_mul_ni(k, acc));
        }
        if (tid == 0) fr_store(&a.sigma[4], fr_add(fr_mul_ni(EB[0], gacc[0]), fr_mul_ni(fr_mul_ni(rp, EB[0]), gacc[1])));
        if (a.r0cells) {
            // the first i-round's linear terms from the parity-split cells (gram.cu), with a(i) = sum_j e_j bit_j:
            //   T_a(0)   = kappa_a sum_j e_j Lin[s][0][0][j]                               (slots 0, 3)
            //   T_c(0)   = kappa_c sum_j e_j Lin[s][0][1][j]                               (slots 1, 4)
            //   T_c(inf) = kappa_c sum_j e_j (Lin[s][1][1] - Lin[s][1][2] - Lin[s][0][2] + Lin[s][0][1])[j]
            // (sum_b E'_c (a(2b+1) - a(2b)) (o(2b+1) - o(2b)) expanded), kappa as the i-round's HI' tables carry
            fr_t (*r0p)[32] = CQ + 4;   // rows 4-9 of the free CQ
            __syncthreads();
            if (tid < 6 * B) {
                const int sl = tid / B, j = tid % B, sw = sl / 3, k = sl % 3;
                const fr_t* L = a.r0cells + 6 * B * sw;
#define R0L(par, q) fr_load(&L[((par) * 3 + (q)) * B + j])
                fr_t v;
                if (k == 0) v = R0L(0, 0);
                else if (k == 1) v = R0L(0, 1);
                else v = fr_add(fr_sub(fr_sub(R0L(1, 1), R0L(1, 2)), R0L(0, 2)), R0L(0, 1));
#undef R0L
                r0p[sl][j] = fr_mul_ni(ej[j], v);
            }
            __syncthreads();
            if (tid < 6) {
                const int sw = tid / 3, k = tid % 3;
                fr_t acc = fr_zero();
                for (int j = 0; j < B; j++) acc = fr_add(acc, r0p[tid][j]);
                const fr_t s = S[0], sp = SP[0];
                const fr_t kap = sw == 0 ? (k == 0 ? fr_mul_ni(r2, s) : fr_mul_ni(r, sp))
                                         : (k == 0 ? fr_mul_ni(fr_mul_ni(rp, r2), s) : fr_mul_ni(fr_mul_ni(rp, r), sp));
                fr_store(&a.r0ext[tid], fr_mul_ni(kap, acc));
            }
        }
    }
    const int nb = (B + 7) / 8;
    for (int e = tid; e < nb * 256; e += blockDim.x) {
        int bb = e >> 8, v = e & 255;
        fr_t acc = fr_zero();
        for (int k = 0; k < 8; k++)
            if (((v >> k) & 1) && 8 * bb + k < B) acc = fr_add(acc, ej[8 * bb + k]);
        fr_store(&a.byte_tab[e], acc);
    }
}

// ---------------------------------------------------------------- i-phase tables
// a0(i) = sum_b T[b][byte_b(Z_i & mask)], a1 likewise from G_A, oms(i) = 1 - sig_i
__global__ void k_relu_materialize(const int32_t* Z, const int32_t* GA, uint64_t D, uint32_t qr_mask, uint32_t sig_bit,
                                   uint32_t nbytes, const fr_t* T, fr_t* a0, fr_t* a1, fr_t* oms) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < D; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t z = (uint32_t)__ldg(Z + i), g = (uint32_t)__ldg(GA + i);
        uint32_t zm = z & qr_mask, gm = g & qr_mask;
        fr_t x = fr_zero(), y = fr_zero();
        for (uint32_t b = 0; b < nbytes; b++) {
            x = fr_add(x, fr_load(&T[b * 256 + ((zm >> (8 * b)) & 255)]));
            y = fr_add(y, fr_load(&T[b * 256 + ((gm >> (8 * b)) & 255)]));
        }
        fr_store(&a0[i], x);
        fr_store(&a1[i], y);
        fr_store(&oms[i], ((z >> sig_bit) & 1) ? fr_zero() : fr_one());
    }
}

struct IRoundArgs {
    uint32_t cpb;          // k_relu_iround_f: CTAs per HI block (grid = 2^hb * cpb)
    const fr_t* src[3];   // a0, a1, oms
    fr_t* dst[3];
    uint64_t n_pairs;
    const fr_t* r_prev;
    const fr_t* lo_cur[5];
    fr_t* lo_next[5];
    fr_t* hi[6];           // scaled HI' tables: Z, A, GA, GZ, b, b' = r' b (rescaled in place by the finalizer)
    uint32_t lo_cnt;       // LO variables of this round (>= 1), including the current one
    uint32_t hb;
    const fr_t* u[5];      // eq points over i (Montgomery)
    uint32_t t;            // i-round index
    fr_t* claim;           // running claim c_t (device); g_t(1) = c_t - g_t(0), then c_{t+1} = g_t(r_t)
    fr_t* partials;
    unsigned int* ticket;
    uint8_t* st;
    uint8_t* msg_out;
    fr_t* r_out;
    uint8_t* point_out;
    // MODE 2 / 3 of k_relu_iround_f: the int32 words (Z, G_A) and the byte table of k_relu_jrounds
    const int32_t* words[2];
    const fr_t* byte_tab;
    uint32_t qr_mask, sig_bit, nbytes;
    // MODE bit 2 (derived X = 1): the per-term running sums (read and updated by the finalizer) and u_x[t]^-1
    fr_t* sigma;
    const fr_t* uinv;
    // MODE bit 3 (round 0 with the linear terms from the bit-sum cells): k_relu_jrounds' six totals, added by the
    // finalizer to slots 0-5
    const fr_t* r0ext;
};

// Finalizer of an i-round (last block, after the grid reduction), in two parts so that the persistent
// kernel can release the next round as soon as r_t exists:
//  iround_transcript: message (g(0), c - g(0), g(2), g(3)) (D4: g(1) follows from g(0) + g(1) = c_t),
//    absorb, squeeze r_t (stored Montgomery at r_out, canonical at point_out); warp 0 only.
//  iround_rescale: HI'_dst = HI'_src * beta(u_x[t], r_t); iround_claim: next claim g_t(r_t) by
//    Lagrange interpolation through 0..3 (every thread calls both).
struct IFinish {
    uint8_t* st;
    fr_t* claim;
    uint8_t* msg_out;
    fr_t* r_out;
    uint8_t* point_out;
    const fr_t* u[5];
    fr_t* hi[6];       // source HI' tables of the round
    fr_t* hi_dst[6];   // rescaled tables (== hi outside the persistent kernel)
    uint32_t t, hb;
};
__device__ __noinline__ void iround_transcript(const IFinish a, const fr_t* g, fr_t* msg /* smem [4] */) {
    __shared__ FsScratch fs;
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        if (lane == 0) {
            msg[0] = g[0];
            msg[1] = fr_sub(fr_load_l2(a.claim), g[0]);
            msg[2] = g[1];
            msg[3] = g[2];
        }
        __syncwarp();
        fs_begin(fs, a.st);
        fs_absorb_frs(fs, "relu/msg", lane < 4 ? msg[lane & 3] : fr_zero(), 4, a.msg_out);
        fr_t rt = fs_challenge(fs, "relu/x");
        if (lane == 0) {
            fr_store(a.r_out, rt);
            fr_canon_to_bytes(fs.rc, a.point_out);
        }
        fs_end(fs, a.st);
    }
    __syncthreads();
}
__device__ __noinline__ void iround_rescale(const IFinish a) {
    __shared__ fr_t eqr[6];
    const int lane = threadIdx.x;
    if (lane < 6) {   // beta(u_x[t], r_t) = 1 - u - r + 2ur, one lane per HI table
        const fr_t rt = fr_load_l2(a.r_out);
        const fr_t* up = lane == 0 ? a.u[0] : lane == 1 ? a.u[1] : lane == 2 ? a.u[2] : lane == 3 ? a.u[3] : a.u[4];
        fr_t u = fr_load(&up[a.t]);
        fr_t ur = fr_mul_cold(u, rt);
        eqr[lane] = fr_add(fr_sub(fr_sub(fr_one(), u), rt), fr_add(ur, ur));
    }
    __syncthreads();
    const uint32_t nh = 1u << a.hb;
    for (uint32_t e = threadIdx.x; e < 6 * nh; e += blockDim.x) {
        uint32_t x = e / nh, hh = e % nh;
        fr_store(&a.hi_dst[x][hh], fr_mul_cold(fr_load_l2(&a.hi[x][hh]), eqr[x]));
    }
}
__device__ __noinline__ void iround_claim(const IFinish a, const fr_t* msg /* smem [4] */) {
    __shared__ fr_t terms[4];
    const int lane = threadIdx.x;
    if (lane < 4) {   // Lagrange term i of g_t(r_t) through 0..3: e_i prod_{j != i}(r - j) / (i - j)
        const fr_t rt = fr_load_l2(a.r_out);
        const int i = lane;
        fr_t num = msg[i];
        for (int j = 0; j < 4; j++)
            if (j != i) num = fr_mul_cold(num, fr_sub(rt, fr_from_u32((uint32_t)j)));
        num = fr_mul_cold(num, (i == 0 || i == 3) ? ZK_INV6 : ZK_INV2);
        terms[i] = (i == 0 || i == 2) ? fr_neg(num) : num;   // denominators -6, 2, -2, 6
    }
    __syncthreads();
    if (lane == 0) fr_store(a.claim, fr_add(fr_add(terms[0], terms[1]), fr_add(terms[2], terms[3])));
}
__device__ __forceinline__ void iround_finish(const IFinish a, const fr_t* g) {
    __shared__ fr_t msg[4];
    iround_transcript(a, g, msg);
    iround_rescale(a);
    iround_claim(a, msg);
}

__device__ __forceinline__ IFinish ifinish_of(const IRoundArgs& a) {
    IFinish f;
    f.st = a.st;
    f.claim = a.claim;
    f.msg_out = a.msg_out;
    f.r_out = a.r_out;
    f.point_out = a.point_out;
    for (int x = 0; x < 5; x++) f.u[x] = a.u[x];
    for (int x = 0; x < 6; x++) f.hi[x] = f.hi_dst[x] = a.hi[x];
    f.t = a.t;
    f.hb = a.hb;
    return f;
}

// Two threads per pair b: side s = 0 carries a0 with E_Z, E_A and the AIVP weight E_b; side s = 1
// carries a1 with E_GA, E_GZ and E_b' = r' E_b (its own HI table, so no per-pair r' product).  Per side
// and X in {0, 2, 3}: P_s(X) = a (E_a + E_c oms) + E_b a (a - 1); X = 1 follows from g(0) + g(1) = c_t.
// (The pre-factoring round kernel, kept as the A/B reference: ZKDL_IROUND_V=0.)
#define IR_MUL fr_mul_ni   // one out-of-line product body: the loop fits the instruction cache
template <bool FOLD>
__global__ void __launch_bounds__(256, 2) k_relu_iround(IRoundArgs a) {
    fr_t acc[3] = {fr_zero(), fr_zero(), fr_zero()};   // X = 0, 2, 3
    const int side = threadIdx.x & 1;
    const uint64_t lo_mask = (1ull << a.lo_cnt) - 1;
    const uint64_t next_count = 1ull << (a.lo_cnt - 1);
    const fr_t* srcA = side ? a.src[1] : a.src[0];
    fr_t* dstA = side ? a.dst[1] : a.dst[0];
    const fr_t* loA = side ? a.lo_cur[2] : a.lo_cur[0];
    const fr_t* loC = side ? a.lo_cur[3] : a.lo_cur[1];
    const fr_t* loB = a.lo_cur[4];
    const fr_t* hiA = side ? a.hi[2] : a.hi[0];
    const fr_t* hiC = side ? a.hi[3] : a.hi[1];
    const fr_t* hiB = side ? a.hi[5] : a.hi[4];
    fr_t r;
    if (FOLD) r = fr_load(a.r_prev);
    const uint64_t first = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 1;
    const uint64_t stride = ((uint64_t)gridDim.x * blockDim.x) >> 1;
    for (uint64_t b = first; b < a.n_pairs; b += stride) {
        fr_t av, ad, om, omd;
        int o0 = 0, od = 0;   // first round: oms(0), oms(1) - oms(0) as small integers (oms is boolean)
        if (FOLD) {
            const fr_t* s = srcA + 4 * b;
            fr_t y0 = fr_load_cg(s), y1 = fr_load_cg(s + 1), y2 = fr_load_cg(s + 2), y3 = fr_load_cg(s + 3);
            fr_t x0 = fr_add(y0, IR_MUL(r, fr_sub(y1, y0)));
            fr_t x1 = fr_add(y2, IR_MUL(r, fr_sub(y3, y2)));
            fr_store(dstA + 2 * b, x0);
            fr_store(dstA + 2 * b + 1, x1);
            av = x0;
            ad = fr_sub(x1, x0);
            // oms fold shared by the pair's two lanes: side s folds entry s and stores it
            const fr_t* so = a.src[2] + 4 * b + 2 * side;
            y0 = fr_load_cg(so);
            y1 = fr_load_cg(so + 1);
            const fr_t mine = fr_add(y0, IR_MUL(r, fr_sub(y1, y0)));
            fr_store(a.dst[2] + 2 * b + side, mine);
            const fr_t other = fr_shfl_xor(mine, 1, __activemask());
            om = side ? other : mine;
            omd = fr_sub(side ? mine : other, om);
        } else {
            av = fr_load_cg(srcA + 2 * b);
            ad = fr_sub(fr_load_cg(srcA + 2 * b + 1), av);
            o0 = !fr_is_zero(fr_load_cg(a.src[2] + 2 * b));
            od = (int)!fr_is_zero(fr_load_cg(a.src[2] + 2 * b + 1)) - o0;
        }
        if (b < next_count) {   // next LO level: side 0 handles Z, A, b; side 1 handles GA, GZ
            fr_store(&a.lo_next[side ? 2 : 0][b], fr_add(fr_load(&loA[2 * b]), fr_load(&loA[2 * b + 1])));
            fr_store(&a.lo_next[side ? 3 : 1][b], fr_add(fr_load(&loC[2 * b]), fr_load(&loC[2 * b + 1])));
            if (side == 0) fr_store(&a.lo_next[4][b], fr_add(fr_load(&loB[2 * b]), fr_load(&loB[2 * b + 1])));
        }
        const uint64_t l0 = (2 * b) & lo_mask;
        const uint64_t h = b >> (a.lo_cnt - 1);
        const fr_t ha = fr_load(&hiA[h]), hc = fr_load(&hiC[h]), hb = fr_load(&hiB[h]);
        fr_t ea = IR_MUL(fr_load(&loA[l0]), ha);
        fr_t ead = fr_sub(IR_MUL(fr_load(&loA[l0 + 1]), ha), ea);
        fr_t ec = IR_MUL(fr_load(&loC[l0]), hc);
        fr_t ecd = fr_sub(IR_MUL(fr_load(&loC[l0 + 1]), hc), ec);
        fr_t eb = IR_MUL(fr_load(&loB[l0]), hb);
        fr_t ebd = fr_sub(IR_MUL(fr_load(&loB[l0 + 1]), hb), eb);
        // P(X) = a (E_a + oms E_c + (a - 1) E_b): three products per evaluation point (two when oms is
        // a small integer in the first round)
#pragma unroll
        for (int X = 0; X < 4; X++) {
            if (X != 1) {
                const fr_t t_c = FOLD ? IR_MUL(ec, om) : fr_mul_small(ec, o0 + X * od);
                const fr_t q = fr_add(fr_add(ea, t_c), IR_MUL(eb, fr_sub(av, fr_one())));
                acc[X == 0 ? 0 : X - 1] = fr_add(acc[X == 0 ? 0 : X - 1], IR_MUL(av, q));
            }
            if (X < 3) {
                av = fr_add(av, ad);
                if (FOLD) om = fr_add(om, omd);
                ea = fr_add(ea, ead);
                ec = fr_add(ec, ecd);
                eb = fr_add(eb, ebd);
            }
        }
    }
    __shared__ fr_t tot[3];
    if (grid_reduce_fr_block<3>(acc, a.partials, a.ticket, tot)) iround_finish(ifinish_of(a), tot);
}

// Factored i-round (default).  The current variable's eq factor is pulled out of every eq table:
// E_x(2b + c) = beta(u_x[t], c) E'_x(b) with E'_x(b) = LO_x[2b] + LO_x[2b+1] (the next LO level, additions
// only: beta(u, 0) + beta(u, 1) = 1) times HI'_x[h] (one value per CTA: every CTA works inside one HI
// block).  Per side the round polynomial is then a sum of three terms, each a fixed linear factor
// beta(u_x[t], X) times a per-pair polynomial that is accumulated on its own:
//   T_a(X) = sum E'_a a(X)                      (linear: accumulated at X = 0, 1)
//   T_c(X) = sum E'_c a(X) oms(X)               (quadratic: X = 0, 1, infinity)
//   T_b(X) = sum E'_b a(X) (a(X) - 1)           (quadratic; both sides' T_b share beta(u_b[t], X))
// with y = E' a formed at X = 0, 1 once (two products) and the quadratic's values at 0, 1, infinity as
// three more (oms is a 0/1 integer in the first round: selects).  That is 15 Fr products per side and
// pair in folding rounds (3 fold + 6 + 3 + 3) and 9 in the first (6 + 3), against 18 and 12 for the
// unfactored form; HI', beta(u_x[t], X) and the cross-side sums are applied once per CTA / per round.
// Values (13 Fr per CTA): Z: T_a side 0 [0..1]; A: T_c side 0 [2..4]; GA: T_a side 1 [5..6];
// GZ: T_c side 1 [7..9]; b: T_b both sides [10..12].
constexpr int IR_NV = 13;

struct IPtrs {   // one side's view of a round (L2 loads: the persistent kernel re-reads buffers it wrote)
    const fr_t* srcA;
    const fr_t* srcO;
    fr_t* dstA;
    fr_t* dstO;
    const fr_t* loA;
    const fr_t* loC;
    const fr_t* loB;
    fr_t* nxA;
    fr_t* nxC;
    fr_t* nxB;   // null on side 1
    // SRC = 1 (rounds 0 and 1 from the int32 words, no materialised tables): this side's word (Z or G_A),
    // the Z words (sign bits), the byte tables in shared memory ([nbytes][256]; round 1: (1 - r_0) T then
    // r_0 T), the masks
    const int32_t* W;
    const int32_t* Zw;
    const fr_t* tb;
    uint32_t qr_mask, sig_bit, nbytes;
};

// i-round input prefetch (ZKDL_IR_PREFETCH): one prefetch.global.L2 per 64-byte piece of the next pair
#ifndef ZKDL_IR_PREFETCH
#define ZKDL_IR_PREFETCH 0
#endif
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
// ZKDL_IR_PF=1 (A/B build): the per-round kernel's fold rounds read through L1 and prefetch the next pair's
// inputs into L1 (the persistent kernel keeps its L2 reads: its tables are written inside the launch)
#ifndef ZKDL_IR_PF
#define ZKDL_IR_PF 0
#endif

// the i-round's three-product groups (ZKDL_IR_MULW): 3 = one three-product body (three interleaved
// chains, ~21 KB of code), 1 = three calls of the single-product body (~7 KB: inside the L0 I-cache)
#ifndef ZKDL_IR_MULW
#define ZKDL_IR_MULW 1
#endif
// the persistent kernel's product groups (its rounds are latency-bound: 3 = one three-chain body per group)
#ifndef ZKDL_IP_MULW
#define ZKDL_IP_MULW 3
#endif
template <int MW = ZKDL_IR_MULW>
__device__ __forceinline__ fr3_t ir_mul3(const fr_t& a0, const fr_t& b0, const fr_t& a1, const fr_t& b1, const fr_t& a2,
                                         const fr_t& b2) {
    if constexpr (MW == 3) {
        return fr_mul3_ni(a0, b0, a1, b1, a2, b2);
    } else if constexpr (MW == 2) {
        const fr2p_t p = fr_mul2_ni(a0, b0, a1, b1);
        return fr3_t{p.x, p.y, fr_mul_ni(a2, b2)};
    } else {
        fr3_t r;
        r.x = fr_mul_ni(a0, b0);
        r.y = fr_mul_ni(a1, b1);
        r.z = fr_mul_ni(a2, b2);
        return r;
    }
}

// a(i) = sum_j beta(r_j, j) bit_j(w_i) as byte-table lookups (the table rows of k_relu_materialize)
__device__ __forceinline__ fr_t byte_sum(const fr_t* tb, uint32_t w, const IPtrs& q) {
    const uint32_t x = w & q.qr_mask;
    fr_t acc = tb[x & 255];
    for (uint32_t k = 1; k < q.nbytes; k++) acc = fr_add(acc, tb[k * 256 + ((x >> (8 * k)) & 255)]);
    return acc;
}

// Accumulate this thread's pairs j = j0, j0 + js, ... < P_blk of HI block h into T[0..7] =
// (T_a(0), T_a(1), T_c(0), T_c(1), T_c(inf), T_b(0), T_b(1), T_b(inf)) of its side.
template <bool FOLD, int SRC = 0, bool DER = false, bool CELLS = false, bool PF = false, int MW = ZKDL_IR_MULW>
__device__ __forceinline__ void iround_pairs(const IPtrs& q, const fr_t& r, uint32_t h, uint32_t pb, uint64_t j0,
                                             uint64_t js, const int side, fr_t (&T)[8]) {
    const fr_t one = fr_one();
    const uint64_t P_blk = 1ull << pb;
    for (uint64_t j = j0; j < P_blk; j += js) {
        const uint64_t b = ((uint64_t)h << pb) + j;
#if ZKDL_IR_PREFETCH
        if (j + js < P_blk) {   // the next pair's inputs into L2 (HBM latency off the loop's critical path)
            const uint64_t bn = b + js;
            if constexpr (SRC == 1 && FOLD) {
                prefetch_l2(reinterpret_cast<const int4*>(q.W) + bn);
                if (side) prefetch_l2(reinterpret_cast<const int4*>(q.Zw) + bn);
            } else if constexpr (SRC == 1) {
                prefetch_l2(reinterpret_cast<const int2*>(q.W) + bn);
                if (side) prefetch_l2(reinterpret_cast<const int2*>(q.Zw) + bn);
            } else if (FOLD) {
                prefetch_l2(q.srcA + 4 * bn);
                prefetch_l2(q.srcA + 4 * bn + 2);
                prefetch_l2(q.srcO + 4 * bn + 2 * side);
            } else {
                prefetch_l2(q.srcA + 2 * bn);
                prefetch_l2(q.srcO + 2 * bn);
            }
        }
#endif
        fr_t a0, a1, om0, om1;
        int o0 = 0, o1 = 0;
        if constexpr (SRC == 1 && FOLD) {
            // round 1 from the words: the fold by r_0 of entries (4b, 4b+1) and (4b+2, 4b+3) is a sum of
            // lookups in (1 - r_0) T and r_0 T; oms folds to 0, 1 - r_0, r_0 or 1
            const int4 w4 = __ldcs(reinterpret_cast<const int4*>(q.W) + b);
            const int4 z4 = side ? __ldcs(reinterpret_cast<const int4*>(q.Zw) + b) : w4;
            const fr_t* t1 = q.tb + q.nbytes * 256;
            a0 = fr_add(byte_sum(q.tb, (uint32_t)w4.x, q), byte_sum(t1, (uint32_t)w4.y, q));
            a1 = fr_add(byte_sum(q.tb, (uint32_t)w4.z, q), byte_sum(t1, (uint32_t)w4.w, q));
            const uint32_t zA = (uint32_t)(side ? z4.z : z4.x), zB = (uint32_t)(side ? z4.w : z4.y);
            const bool oA = !((zA >> q.sig_bit) & 1), oB = !((zB >> q.sig_bit) & 1);
            const fr_t mine = oA ? (oB ? fr_one() : fr_sub(fr_one(), r)) : (oB ? r : fr_zero());
            fr_store(q.dstA + 2 * b, a0);
            fr_store(q.dstA + 2 * b + 1, a1);
            fr_store(q.dstO + 2 * b + side, mine);
            const fr_t other = fr_shfl_xor(mine, 1, __activemask());
            om0 = side ? other : mine;
            om1 = side ? mine : other;
        } else if constexpr (SRC == 1) {   // round 0 from the words
            const int2 w2 = __ldcs(reinterpret_cast<const int2*>(q.W) + b);
            const int2 z2 = side ? __ldcs(reinterpret_cast<const int2*>(q.Zw) + b) : w2;
            a0 = byte_sum(q.tb, (uint32_t)w2.x, q);
            a1 = byte_sum(q.tb, (uint32_t)w2.y, q);
            o0 = !(((uint32_t)z2.x >> q.sig_bit) & 1);
            o1 = !(((uint32_t)z2.y >> q.sig_bit) & 1);
        } else if (FOLD) {
            const fr_t* s = q.srcA + 4 * b;
            // oms fold shared by the pair's two lanes: side s folds entry s and stores it
            const fr_t* so = q.srcO + 4 * b + 2 * side;
            fr_t y0, y1, y2, y3, z0, z1;
            if constexpr (PF) {
                if (j + js < P_blk) {   // the next pair's inputs into L1
                    prefetch_l1(s + 4 * js);
                    prefetch_l1(so + 4 * js);
                    prefetch_l1(&q.loA[2 * (j + js)]);
                    prefetch_l1(&q.loC[2 * (j + js)]);
                    prefetch_l1(&q.loB[2 * (j + js)]);
                }
                y0 = fr_load(s); y1 = fr_load(s + 1); y2 = fr_load(s + 2); y3 = fr_load(s + 3);
                z0 = fr_load(so); z1 = fr_load(so + 1);
            } else {
                y0 = fr_load_l2(s); y1 = fr_load_l2(s + 1); y2 = fr_load_l2(s + 2); y3 = fr_load_l2(s + 3);
                z0 = fr_load_l2(so); z1 = fr_load_l2(so + 1);
            }
            const fr3_t f = ir_mul3<MW>(r, fr_sub(y1, y0), r, fr_sub(y3, y2), r, fr_sub(z1, z0));
            a0 = fr_add(y0, f.x);
            a1 = fr_add(y2, f.y);
            const fr_t mine = fr_add(z0, f.z);
            fr_store(q.dstA + 2 * b, a0);
            fr_store(q.dstA + 2 * b + 1, a1);
            fr_store(q.dstO + 2 * b + side, mine);
            const fr_t other = fr_shfl_xor(mine, 1, __activemask());
            om0 = side ? other : mine;
            om1 = side ? mine : other;
        } else {
            a0 = fr_load_cg(q.srcA + 2 * b);
            a1 = fr_load_cg(q.srcA + 2 * b + 1);
            o0 = !fr_is_zero(fr_load_cg(q.srcO + 2 * b));
            o1 = !fr_is_zero(fr_load_cg(q.srcO + 2 * b + 1));
        }
        const fr_t eB = PF ? fr_add(fr_load(&q.loB[2 * j]), fr_load(&q.loB[2 * j + 1]))
                           : fr_add(fr_load_l2(&q.loB[2 * j]), fr_load_l2(&q.loB[2 * j + 1]));
        if constexpr (CELLS) {   // the linear terms come from the bit-sum cells: only the binary check here
            if (h == 0) {   // the next LO level: side 0 writes Z, A, b; side 1 writes GA, GZ
                fr_store(&q.nxA[j], fr_add(fr_load_l2(&q.loA[2 * j]), fr_load_l2(&q.loA[2 * j + 1])));
                fr_store(&q.nxC[j], fr_add(fr_load_l2(&q.loC[2 * j]), fr_load_l2(&q.loC[2 * j + 1])));
                if (q.nxB) fr_store(&q.nxB[j], eB);
            }
            const fr_t dA = fr_sub(a1, a0);
            const fr_t zB0 = fr_mul_ni(eB, a0), zD = fr_mul_ni(eB, dA);
            T[3] = fr_add(T[3], fr_mul_ni(zB0, fr_sub(a0, one)));
            T[4] = fr_add(T[4], fr_mul_ni(zD, dA));
            (void)o0;
            (void)o1;
            (void)om0;
            (void)om1;
            continue;
        }
        const fr_t eA = PF ? fr_add(fr_load(&q.loA[2 * j]), fr_load(&q.loA[2 * j + 1]))
                           : fr_add(fr_load_l2(&q.loA[2 * j]), fr_load_l2(&q.loA[2 * j + 1]));
        const fr_t eC = PF ? fr_add(fr_load(&q.loC[2 * j]), fr_load(&q.loC[2 * j + 1]))
                           : fr_add(fr_load_l2(&q.loC[2 * j]), fr_load_l2(&q.loC[2 * j + 1]));
        if (h == 0) {   // the next LO level: side 0 writes Z, A, b; side 1 writes GA, GZ
            fr_store(&q.nxA[j], eA);
            fr_store(&q.nxC[j], eC);
            if (q.nxB) fr_store(&q.nxB[j], eB);
        }
        if constexpr (DER) {
            // derived X = 1 (the finalizer gets T_x(1) from the running per-term sum): T_a(0), T_c(0),
            // T_c(inf) = sum e_C (a1 - a0)(oms1 - oms0), T_b(0), T_b(inf) = sum e_b (a1 - a0)^2 into T[0..4]
            const fr_t dA = fr_sub(a1, a0);
            const fr_t tA = fr_mul_ni(eA, a0);
            const fr_t yC0 = fr_mul_ni(eC, a0), yD = fr_mul_ni(eC, dA);
            const fr_t zB0 = fr_mul_ni(eB, a0), zD = fr_mul_ni(eB, dA);
            T[0] = fr_add(T[0], tA);
            if (FOLD) {
                T[1] = fr_add(T[1], fr_mul_ni(yC0, om0));
                T[2] = fr_add(T[2], fr_mul_ni(yD, fr_sub(om1, om0)));
            } else {   // oms in {0, 1}
                const fr_t zero = fr_zero();
                T[1] = fr_add(T[1], o0 ? yC0 : zero);
                T[2] = fr_add(T[2], o1 == o0 ? zero : (o1 ? yD : fr_neg(yD)));
            }
            T[3] = fr_add(T[3], fr_mul_ni(zB0, fr_sub(a0, one)));
            T[4] = fr_add(T[4], fr_mul_ni(zD, dA));
            continue;
        }
        const fr3_t p = ir_mul3<MW>(eA, a0, eA, a1, eC, a0);
        const fr3_t pq = ir_mul3<MW>(eC, a1, eB, a0, eB, a1);
        T[0] = fr_add(T[0], p.x);
        T[1] = fr_add(T[1], p.y);
        const fr_t yC0 = p.z, yC1 = pq.x, zB0 = pq.y, zB1 = pq.z;
        if (FOLD) {
            const fr3_t c = ir_mul3<MW>(yC0, om0, yC1, om1, fr_sub(yC1, yC0), fr_sub(om1, om0));
            T[2] = fr_add(T[2], c.x);
            T[3] = fr_add(T[3], c.y);
            T[4] = fr_add(T[4], c.z);
        } else {   // oms(0), oms(1) in {0, 1}: T_c at infinity is (o1 - o0)(y1 - y0)
            const fr_t yd = fr_sub(yC1, yC0);
            const fr_t zero = fr_zero();
            T[2] = fr_add(T[2], o0 ? yC0 : zero);
            T[3] = fr_add(T[3], o1 ? yC1 : zero);
            T[4] = fr_add(T[4], o1 == o0 ? zero : (o1 ? yd : fr_neg(yd)));
        }
        const fr3_t d = ir_mul3<MW>(zB0, fr_sub(a0, one), zB1, fr_sub(a1, one), fr_sub(zB1, zB0), fr_sub(a1, a0));
        T[5] = fr_add(T[5], d.x);
        T[6] = fr_add(T[6], d.y);
        T[7] = fr_add(T[7], d.z);
    }
}

// T[] times this CTA's HI' values (kappa_x * prior betas; side 1's b table carries r'), then scattered
// into the 13 reduction slots (zeros in the other side's slots).  Threads without pairs skip the products.
__device__ __forceinline__ void iround_scale_scatter(fr_t (&T)[8], fr_t* const* hi, uint32_t h, int side, bool any,
                                                     fr_t (&acc)[16]) {
    if (any) {
        const fr_t hA = fr_load_l2(&(side ? hi[2] : hi[0])[h]);
        const fr_t hC = fr_load_l2(&(side ? hi[3] : hi[1])[h]);
        const fr_t hB = fr_load_l2(&(side ? hi[5] : hi[4])[h]);
        const fr3_t u = fr_mul3_ni(T[0], hA, T[1], hA, T[2], hC);
        const fr3_t v = fr_mul3_ni(T[3], hC, T[4], hC, T[5], hB);
        const fr3_t w = fr_mul3_ni(T[6], hB, T[7], hB, fr_zero(), fr_zero());
        T[0] = u.x; T[1] = u.y; T[2] = u.z; T[3] = v.x; T[4] = v.y; T[5] = v.z; T[6] = w.x; T[7] = w.y;
    }
    const fr_t zero = fr_zero();
#pragma unroll
    for (int k = 0; k < 5; k++) {
        acc[k] = side ? zero : T[k];
        acc[5 + k] = side ? T[k] : zero;
    }
    acc[10] = T[5];
    acc[11] = T[6];
    acc[12] = T[7];
    acc[13] = acc[14] = acc[15] = zero;
}

// The derived-X=1 layout: T[0..4] = (T_a(0), T_c(0), T_c(inf), T_b(0), T_b(inf)) of a side, times HI'; slots
// 0 = Z, 1-2 = A, 3 = GA, 4-5 = GZ (the side's), 6-7 = b (both sides)
constexpr int IR_NV_DER = 8;
__device__ __forceinline__ void iround_scale_scatter_der(fr_t (&T)[8], fr_t* const* hi, uint32_t h, int side, bool any,
                                                         fr_t (&acc)[16]) {
    if (any) {
        const fr_t hA = fr_load_l2(&(side ? hi[2] : hi[0])[h]);
        const fr_t hC = fr_load_l2(&(side ? hi[3] : hi[1])[h]);
        const fr_t hB = fr_load_l2(&(side ? hi[5] : hi[4])[h]);
        T[0] = fr_mul_ni(T[0], hA);
        T[1] = fr_mul_ni(T[1], hC);
        T[2] = fr_mul_ni(T[2], hC);
        T[3] = fr_mul_ni(T[3], hB);
        T[4] = fr_mul_ni(T[4], hB);
    }
    const fr_t zero = fr_zero();
#pragma unroll
    for (int k = 0; k < 3; k++) {
        acc[k] = side ? zero : T[k];
        acc[3 + k] = side ? T[k] : zero;
    }
    acc[6] = T[3];
    acc[7] = T[4];
#pragma unroll
    for (int k = 8; k < 16; k++) acc[k] = zero;
}

// Transposed block reduction of 16 values per thread: each butterfly step of the warp halves the
// values a lane keeps (16 Fr shuffles and 16 additions per lane instead of 16 x 5 of a per-value
// tree), then warp 0 adds the 8 warps' rows.  On return lane k < 16 of warp 0 holds the total of
// value k in v[0] (the other lanes hold partial sums).  Small code, short dependency chains: this
// runs once per round on the critical path.
__device__ __forceinline__ void warp_transpose_sum16(fr_t (&v)[16]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 16, c = 8; o >= 2; o >>= 1, c >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int i = 0; i < c; i++) {
            fr_t send, keep;
#pragma unroll
            for (int l = 0; l < 8; l++) {
                send.v[l] = up ? v[i].v[l] : v[i + c].v[l];
                keep.v[l] = up ? v[i + c].v[l] : v[i].v[l];
            }
            v[i] = fr_add(keep, fr_shfl_xor(send, o));
        }
    }
    v[0] = fr_add(v[0], fr_shfl_xor(v[0], 1));   // lane holds the warp total of value (lane >> 1) & 15
}
__device__ __forceinline__ void block_transpose_sum16(fr_t (&v)[16], fr_t* sm /* >= 8 * 16 */) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    warp_transpose_sum16(v);
    if (!(lane & 1)) sm[wid * 16 + (lane >> 1)] = v[0];
    __syncthreads();
    if (wid == 0 && lane < 16) {
        fr_t x = sm[lane];
        for (int w = 1; w < nw; w++) x = fr_add(x, sm[w * 16 + lane]);
        v[0] = x;
    }
    __syncthreads();
}

// g(X) = sum_x beta(u_x[t], X) T_x(X) at X = 0, 2, 3 from the 13 round totals (lane 3x + k, X = {0,2,3}[k]);
// called by every thread of the block, writes g[0..2].
__device__ __noinline__ void iround_g(const fr_t* tot, const fr_t* const* u, uint32_t t, fr_t* prod, fr_t* g) {
    const int lane = threadIdx.x;
    const fr_t one = fr_one(), zero = fr_zero();
    if (lane < 15) {
        const int x = lane / 3, k = lane % 3;
        const uint32_t X = k == 0 ? 0u : k + 1u;
        const int base = x == 0 ? 0 : x == 1 ? 2 : x == 2 ? 5 : x == 3 ? 7 : 10;
        const bool quad = x != 0 && x != 2;
        const fr_t V0 = tot[base], V1 = tot[base + 1], Vi = quad ? tot[base + 2] : zero;
        // T(X) = V0 + X (V1 - V0 - Vi) + X^2 Vi
        const fr_t lin = fr_sub(fr_sub(V1, V0), Vi);
        fr_t T = V0;
        for (uint32_t i = 0; i < X; i++) T = fr_add(T, lin);
        for (uint32_t i = 0; i < X * X; i++) T = fr_add(T, Vi);
        // beta(u, X) = (1 - u) + X (2u - 1)
        const fr_t uu = fr_load(&u[x][t]);
        const fr_t slope = fr_sub(fr_add(uu, uu), one);
        fr_t be = fr_sub(one, uu);
        for (uint32_t i = 0; i < X; i++) be = fr_add(be, slope);
        prod[lane] = fr_mul_cold(be, T);
    }
    __syncthreads();
    if (lane < 3) {
        fr_t sum = zero;
        for (int x = 0; x < 5; x++) sum = fr_add(sum, prod[3 * x + lane]);
        g[lane] = sum;
    }
    __syncthreads();
}

// Derived X = 1 (MODE bit 2): per term x the round's totals V0 = T_x(0) (and V_inf for the quadratic terms)
// come from the pairs; T_x(1) follows from the term's running sum sigma_x = beta(u, 0) T_x(0) + beta(u, 1) T_x(1):
//     T_x(1) = (sigma_x - (1 - u) V0) u^-1                      (u = u_x[t], its inverse precomputed)
// and g(X) = sum_x beta(u_x[t], X) T_x(X) as in iround_g.  After r_t: sigma_x <- beta(u_x[t], r_t) T_x(r_t).
// (The proof is the same bytes: the three-value form of every term is the one the explicit path sums.)
__device__ __noinline__ void iround_g_der(const fr_t* tot, const fr_t* const* u, uint32_t t, const fr_t* sigma,
                                          const fr_t* uinv, fr_t* V /* smem [15] */, fr_t* prod, fr_t* g) {
    const int lane = threadIdx.x;
    if (lane < 5) {
        const int x = lane, base = x == 0 ? 0 : x == 1 ? 1 : x == 2 ? 3 : x == 3 ? 4 : 6;
        const bool quad = x != 0 && x != 2;
        const fr_t V0 = tot[base], Vi = quad ? tot[base + 1] : fr_zero();
        const fr_t uu = fr_load(&u[x][t]);
        const fr_t V1 = fr_mul_cold(fr_sub(fr_load_l2(&sigma[x]), fr_mul_cold(fr_sub(fr_one(), uu), V0)), fr_load(&uinv[x]));
        V[3 * x] = V0;
        V[3 * x + 1] = V1;
        V[3 * x + 2] = Vi;
    }
    __syncthreads();
    const fr_t one = fr_one(), zero = fr_zero();
    if (lane < 15) {
        const int x = lane / 3, k = lane % 3;
        const uint32_t X = k == 0 ? 0u : k + 1u;
        const fr_t V0 = V[3 * x], V1 = V[3 * x + 1], Vi = V[3 * x + 2];
        const fr_t lin = fr_sub(fr_sub(V1, V0), Vi);
        fr_t T = V0;
        for (uint32_t i = 0; i < X; i++) T = fr_add(T, lin);
        for (uint32_t i = 0; i < X * X; i++) T = fr_add(T, Vi);
        const fr_t uu = fr_load(&u[x][t]);
        const fr_t slope = fr_sub(fr_add(uu, uu), one);
        fr_t be = fr_sub(one, uu);
        for (uint32_t i = 0; i < X; i++) be = fr_add(be, slope);
        prod[lane] = fr_mul_cold(be, T);
    }
    __syncthreads();
    if (lane < 3) {
        fr_t sum = zero;
        for (int x = 0; x < 5; x++) sum = fr_add(sum, prod[3 * x + lane]);
        g[lane] = sum;
    }
    __syncthreads();
}
// sigma_x <- beta(u_x[t], r_t) T_x(r_t) (lanes 0-4, after r_t is published)
__device__ __noinline__ void iround_sigma_der(const fr_t* V, const fr_t* const* u, uint32_t t, const fr_t* r_t, fr_t* sigma) {
    const int x = threadIdx.x;
    if (x < 5) {
        const fr_t r = fr_load_l2(r_t), uu = fr_load(&u[x][t]);
        const fr_t V0 = V[3 * x], V1 = V[3 * x + 1], Vi = V[3 * x + 2];
        const fr_t lin = fr_sub(fr_sub(V1, V0), Vi);
        const fr_t Tr = fr_add(fr_add(V0, fr_mul_cold(r, lin)), fr_mul_cold(fr_mul_cold(r, r), Vi));
        const fr_t ur = fr_mul_cold(uu, r);
        const fr_t be = fr_add(fr_sub(fr_sub(fr_one(), uu), r), fr_add(ur, ur));
        fr_store(&sigma[x], fr_mul_cold(be, Tr));
    }
}

// u^-1 for the derived-X=1 rounds: out[t][x] = u_x[t]^-1, t < t1 (Fermat; traps on u = 0, probability ~2^-250
// per value, rather than emit a wrong proof)
struct UPts {
    const fr_t* u[5];
};
// one value per warp (lane 0): the binary GCD's data-dependent loops would serialise a warp's lanes
__global__ void k_relu_uinv(UPts P, uint32_t t1, fr_t* out) {
    const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= 5 * t1 || (threadIdx.x & 31)) return;
    const uint32_t t = i / 5, x = i % 5;
    const fr_t u = fr_load(&P.u[x][t]);
    if (fr_is_zero(u)) __trap();
    fr_store(&out[i], fr_inv_bgcd(u));
}

// MODE: bit 0 = FOLD, bit 1 = SRC (rounds 0 / 1 from the int32 words through byte tables in shared memory),
// bit 2 = DER (the X = 1 totals derived from the per-term sums), bit 3 = CELLS (round 0 only, with DER: the
// linear terms T_a(0), T_c(0), T_c(inf) from the bit-sum cells, k_relu_jrounds' r0ext; the pairs sum the binary
// check only)
template <int MODE>
// the factored i-round's CTA shape (threads, CTAs per SM): registers per thread = 64K / (threads x CTAs)
#ifndef ZKDL_IR_LB_T
#define ZKDL_IR_LB_T 256
#endif
#ifndef ZKDL_IR_LB_B
#define ZKDL_IR_LB_B 2
#endif
__global__ void __launch_bounds__(ZKDL_IR_LB_T, ZKDL_IR_LB_B) k_relu_iround_f(IRoundArgs a) {
    constexpr bool FOLD = MODE & 1;
    constexpr int SRC = (MODE >> 1) & 1;
    constexpr bool DER = MODE & 4;
    constexpr bool CELLS = MODE & 8;
    static_assert(!CELLS || (DER && !FOLD), "CELLS: the first (derived) round only");
    constexpr int NV = DER ? IR_NV_DER : IR_NV;
    const int side = threadIdx.x & 1;
    const uint32_t pb = a.lo_cnt - 1;   // log2 of the pairs per HI block
    const uint32_t h = blockIdx.x / a.cpb, cib = blockIdx.x % a.cpb;
    IPtrs q;
    q.srcA = side ? a.src[1] : a.src[0];
    q.srcO = a.src[2];
    q.dstA = side ? a.dst[1] : a.dst[0];
    q.dstO = a.dst[2];
    q.loA = side ? a.lo_cur[2] : a.lo_cur[0];
    q.loC = side ? a.lo_cur[3] : a.lo_cur[1];
    q.loB = a.lo_cur[4];
    q.nxA = a.lo_next[side ? 2 : 0];
    q.nxC = a.lo_next[side ? 3 : 1];
    q.nxB = side ? nullptr : a.lo_next[4];
    fr_t r;
    if (FOLD) r = fr_load(a.r_prev);
    if constexpr (SRC == 1) {   // byte tables into shared memory (round 1: scaled by 1 - r_0 and r_0)
        extern __shared__ fr_t tbs[];
        const uint32_t n = a.nbytes * 256;
        const fr_t omr = fr_sub(fr_one(), r);
        for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) {
            const fr_t v = fr_load(&a.byte_tab[e]);
            if (FOLD) {
                tbs[e] = fr_mul_ni(v, omr);
                tbs[n + e] = fr_mul_ni(v, r);
            } else {
                tbs[e] = v;
            }
        }
        __syncthreads();
        q.W = side ? a.words[1] : a.words[0];
        q.Zw = a.words[0];
        q.tb = tbs;
        q.qr_mask = a.qr_mask;
        q.sig_bit = a.sig_bit;
        q.nbytes = a.nbytes;
    }
    fr_t T[8];
#pragma unroll
    for (int k = 0; k < 8; k++) T[k] = fr_zero();
    const uint64_t j0 = (uint64_t)cib * (blockDim.x >> 1) + (threadIdx.x >> 1);
    iround_pairs<FOLD, SRC, DER, CELLS, ZKDL_IR_PF != 0 && FOLD && SRC == 0>(q, r, h, pb, j0,
                                                                            (uint64_t)a.cpb * (blockDim.x >> 1), side, T);
    fr_t v[16];
    if constexpr (DER)
        iround_scale_scatter_der(T, a.hi, h, side, j0 < (1ull << pb), v);
    else
        iround_scale_scatter(T, a.hi, h, side, j0 < (1ull << pb), v);
    __shared__ fr_t sm[8 * 16];
    __shared__ fr_t tot[16];
    __shared__ fr_t prod[15];
    __shared__ fr_t g[3];
    __shared__ bool is_last;
    block_transpose_sum16(v, sm);
    if (threadIdx.x < NV) fr_store(&a.partials[blockIdx.x * NV + threadIdx.x], v[0]);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        is_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    {   // thread i sums the partials of CTAs i, i + 256, ...
        fr_t w[16];
#pragma unroll
        for (int k = 0; k < 16; k++) w[k] = fr_zero();
        for (unsigned int bb = threadIdx.x; bb < gridDim.x; bb += blockDim.x)
#pragma unroll
            for (int k = 0; k < NV; k++) w[k] = fr_add(w[k], fr_load_l2(&a.partials[bb * NV + k]));
        block_transpose_sum16(w, sm);
        if (threadIdx.x < NV) tot[threadIdx.x] = w[0];
        if constexpr (CELLS) {
            if (threadIdx.x < 6) tot[threadIdx.x] = fr_add(tot[threadIdx.x], fr_load_l2(&a.r0ext[threadIdx.x]));
        }
    }
    if (threadIdx.x == 0) *a.ticket = 0;
    __syncthreads();
    if constexpr (DER) {
        __shared__ fr_t V[15];
        __shared__ fr_t msg[4];
        iround_g_der(tot, a.u, a.t, a.sigma, a.uinv, V, prod, g);
        const IFinish f = ifinish_of(a);
        iround_transcript(f, g, msg);
        iround_rescale(f);
        iround_claim(f, msg);
        iround_sigma_der(V, a.u, a.t, a.r_out, a.sigma);
    } else {
        iround_g(tot, a.u, a.t, prod, g);
        iround_finish(ifinish_of(a), g);
    }
}

// The small i-rounds t0 .. t1-1 in ONE cooperative launch (1 + 2^hb * cpb CTAs, at most one per SM):
// per round the workers fold, accumulate, reduce and publish their 13 partials and bump a monotonic
// arrival counter; block 0 (dedicated) sums them, forms g, runs the transcript step and releases the
// next round through `flag` as soon as r_t exists; the claim update and the HI' rescale (into the other
// HI' buffer) follow off the critical path and are released through `hiflag`, which the workers
// only need after their pair loop.  Every buffer written inside the launch is read back through L2
// (ld.cg): L1 is not coherent across SMs.  The code stays in the instruction cache across rounds.
struct IPersistArgs {
    const fr_t* full[3];    // sources of round 1 (round 0 does not fold)
    fr_t* buf[2][3];        // round t folds into buf[t & 1]
    fr_t* LO[5][2];         // round t reads LO[x][t & 1] and writes LO[x][(t & 1) ^ 1]
    fr_t* hi[2][6];         // round t reads hi[(t - t0) & 1] and writes the rescaled tables to the other
    const fr_t* u[5];
    uint32_t t0, t1, H, hb, cpb;
    fr_t* claim;
    fr_t* r_i;              // r of i-round t at r_i[t]
    uint8_t* msg_base;      // i-round t message at msg_base + 128 t
    uint8_t* point_base;    // r_t canonical at point_base + 32 t
    uint8_t* st;
    fr_t* partials;         // (gridDim.x - 1) * 13
    unsigned int* arrive;
    unsigned int* flag;     // rounds whose r_t is published
    unsigned int* hiflag;   // rounds whose HI' rescale is published
    unsigned long long* trace;   // diagnostics (ZKDL_IPERSIST_TRACE): 4 timestamps per round, or null
    // DER (derived X = 1, as k_relu_iround_f MODE bit 2): the per-term running sums and u_x[t]^-1 (5 per round)
    fr_t* sigma;
    const fr_t* uinv;
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned int ld_volatile_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void wait_counter(const unsigned int* p, unsigned int target) {
    if (threadIdx.x == 0) {
        while (ld_volatile_u32(p) < target) __nanosleep(64);
        __threadfence();
    }
    __syncthreads();
}

template <bool DER>
__global__ void __launch_bounds__(256, 2) k_relu_ipersist(IPersistArgs a) {
    constexpr int NV = DER ? IR_NV_DER : IR_NV;
    __shared__ fr_t sm[8 * 16];
    __shared__ fr_t tot[16];
    __shared__ fr_t prod[15];
    __shared__ fr_t g[3];
    __shared__ fr_t msg[4];
    const int side = threadIdx.x & 1;
    const uint32_t nworkers = gridDim.x - 1;
    for (uint32_t t = a.t0; t < a.t1; t++) {
        const uint32_t pb = a.H - t - 1;
        const int lv = t & 1, hv = (t - a.t0) & 1;
        if (blockIdx.x != 0) {
            if (t > a.t0) wait_counter(a.flag, t);   // r_{t-1}, the LO level and the folded tables
            unsigned long long* wtr = (a.trace && blockIdx.x == 1 && threadIdx.x == 0) ? a.trace + 4ull * (a.t1 - a.t0) + 4ull * (t - a.t0) : nullptr;
            if (wtr) wtr[0] = globaltimer_ns();
            const uint32_t w = blockIdx.x - 1, h = w / a.cpb, cib = w % a.cpb;
            IPtrs q;
            const fr_t* const* src = t == 1 ? a.full : (const fr_t* const*)a.buf[(t - 1) & 1];
            q.srcA = side ? src[1] : src[0];
            q.srcO = src[2];
            q.dstA = side ? a.buf[t & 1][1] : a.buf[t & 1][0];
            q.dstO = a.buf[t & 1][2];
            q.loA = side ? a.LO[2][lv] : a.LO[0][lv];
            q.loC = side ? a.LO[3][lv] : a.LO[1][lv];
            q.loB = a.LO[4][lv];
            q.nxA = a.LO[side ? 2 : 0][lv ^ 1];
            q.nxC = a.LO[side ? 3 : 1][lv ^ 1];
            q.nxB = side ? nullptr : a.LO[4][lv ^ 1];
            const fr_t r = fr_load_l2(&a.r_i[t - 1]);
            fr_t T[8];
#pragma unroll
            for (int k = 0; k < 8; k++) T[k] = fr_zero();
            const uint64_t j0 = (uint64_t)cib * (blockDim.x >> 1) + (threadIdx.x >> 1);
            // the latency-bound rounds: three interleaved product chains per call (one call's latency for the
            // three independent products of a step, instead of three calls in sequence)
            iround_pairs<true, 0, DER, false, false, ZKDL_IP_MULW>(q, r, h, pb, j0, (uint64_t)a.cpb * (blockDim.x >> 1),
                                                                  side, T);
            if (wtr) wtr[1] = globaltimer_ns();
            if (t > a.t0) wait_counter(a.hiflag, t);   // HI' rescaled by round t-1
            if (wtr) wtr[2] = globaltimer_ns();
            fr_t v[16];
            if constexpr (DER)
                iround_scale_scatter_der(T, a.hi[hv], h, side, j0 < (1ull << pb), v);
            else
                iround_scale_scatter(T, a.hi[hv], h, side, j0 < (1ull << pb), v);
            block_transpose_sum16(v, sm);
            if (threadIdx.x < NV) fr_store(&a.partials[w * NV + threadIdx.x], v[0]);
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(a.arrive, 1u);
                if (wtr) wtr[3] = globaltimer_ns();
            }
        } else {
            wait_counter(a.arrive, (t - a.t0 + 1) * nworkers);
            if (a.trace && threadIdx.x == 0) a.trace[(t - a.t0) * 4 + 0] = globaltimer_ns();
            {
                fr_t v[16];
#pragma unroll
                for (int k = 0; k < 16; k++) v[k] = fr_zero();
                for (unsigned int bb = threadIdx.x; bb < nworkers; bb += blockDim.x)
#pragma unroll
                    for (int k = 0; k < NV; k++) v[k] = fr_add(v[k], fr_load_l2(&a.partials[bb * NV + k]));
                block_transpose_sum16(v, sm);
                if (threadIdx.x < NV) tot[threadIdx.x] = v[0];
            }
            __syncthreads();
            if (a.trace && threadIdx.x == 0) a.trace[(t - a.t0) * 4 + 1] = globaltimer_ns();
            __shared__ fr_t Vd[15];
            if constexpr (DER)
                iround_g_der(tot, a.u, t, a.sigma, a.uinv + 5ull * t, Vd, prod, g);
            else
                iround_g(tot, a.u, t, prod, g);
            IFinish f;
            f.st = a.st;
            f.claim = a.claim;
            f.msg_out = a.msg_base + 128ull * t;
            f.r_out = a.r_i + t;
            f.point_out = a.point_base + 32ull * t;
            for (int x = 0; x < 5; x++) f.u[x] = a.u[x];
            for (int x = 0; x < 6; x++) {
                f.hi[x] = a.hi[hv][x];
                f.hi_dst[x] = a.hi[hv ^ 1][x];
            }
            f.t = t;
            f.hb = a.hb;
            iround_transcript(f, g, msg);
            if (threadIdx.x == 0) {
                __threadfence();
                atomicExch(a.flag, t + 1);
                if (a.trace) a.trace[(t - a.t0) * 4 + 2] = globaltimer_ns();
            }
            iround_rescale(f);
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                atomicExch(a.hiflag, t + 1);
                if (a.trace) a.trace[(t - a.t0) * 4 + 3] = globaltimer_ns();
            }
            iround_claim(f, msg);   // needed only by the next round's message
            if constexpr (DER) iround_sigma_der(Vd, a.u, t, a.r_i + t, a.sigma);
        }
    }
}

// Last hb i-rounds in one CTA with every table (a0, a1, oms, 5 eq) materialised in shared memory.
struct ITailArgs {
    const fr_t* src[3];
    int fold;               // fold src (2 * n0 entries) by r_prev first
    const fr_t* r_prev;
    const fr_t* hi[5];      // E_x tables (n0 entries, already scaled)
    uint32_t hb;            // rounds in the tail; n0 = 2^hb
    const fr_t* kappa;
    uint8_t* st;
    uint8_t* msg_out;       // hb x 128 bytes
    uint8_t* point_out;     // hb x 32
    fr_t* r_out;
    uint8_t* finals_out;    // 96 bytes
};

__global__ void __launch_bounds__(256) k_relu_itail(ITailArgs a) {
    __shared__ fr_t T[8][32];
    __shared__ fr_t vals[16][4];
    __shared__ fr_t rt_sm;
    const int tid = threadIdx.x;
    const int n0 = 1 << a.hb;
    const fr_t rp = fr_load(&a.kappa[5]);
    for (int e = tid; e < 3 * n0; e += blockDim.x) {
        int k = e / n0, i = e % n0;
        fr_t v;
        if (a.fold) {
            fr_t r = fr_load(a.r_prev);
            fr_t y0 = fr_load(&a.src[k][2 * i]), y1 = fr_load(&a.src[k][2 * i + 1]);
            v = fr_add(y0, fr_mul_cold(r, fr_sub(y1, y0)));
        } else {
            v = fr_load(&a.src[k][i]);
        }
        T[k][i] = v;
    }
    for (int e = tid; e < 5 * n0; e += blockDim.x) T[3 + e / n0][e % n0] = fr_load(&a.hi[e / n0][e % n0]);
    __shared__ FsScratch fs;
    if (tid < 32) fs_begin(fs, a.st);
    __syncthreads();
    for (uint32_t t = 0; t < a.hb; t++) {
        const int n = n0 >> t, np = n >> 1;
        if (tid < 4 * np) {
            const int b = tid >> 2, X = tid & 3;
            // v(X) = T(2b) + X (T(2b+1) - T(2b)) for X in 0..3: additions only
            fr_t v[8];
            for (int k = 0; k < 8; k++) {
                const fr_t y0 = T[k][2 * b], y1 = T[k][2 * b + 1], d = fr_sub(y1, y0);
                v[k] = X == 0 ? y0 : X == 1 ? y1 : X == 2 ? fr_add(y1, d) : fr_add(fr_add(y1, d), d);
            }
            // tables: 0 a0, 1 a1, 2 oms, 3 EZ, 4 EA, 5 EGA, 6 EGZ, 7 Eb; independent products grouped in threes
            // (latency: this single-CTA kernel is on the critical path)
            const fr_t one = fr_one();
            const fr3_t l1 = fr_mul3_ni(v[4], v[2], v[6], v[2], v[0], fr_sub(v[0], one));
            const fr_t l1b = fr_mul_ni(v[1], fr_sub(v[1], one));
            const fr3_t l2 = fr_mul3_ni(v[0], fr_add(v[3], l1.x), v[1], fr_add(v[5], l1.y), rp, l1b);
            const fr_t q = fr_add(l1.z, l2.z);
            vals[b][X] = fr_add(fr_add(l2.x, l2.y), fr_mul_ni(v[7], q));
        }
        __syncthreads();
        if (tid < 32) {
            fr_t ev = fr_zero();
            if (tid < 4)
                for (int b = 0; b < np; b++) ev = fr_add(ev, vals[b][tid]);
            fs_absorb_frs(fs, "relu/msg", ev, 4, a.msg_out + 128ull * t);
            fr_t rt = fs_challenge(fs, "relu/x");
            if (tid == 0) {
                fr_store(&a.r_out[t], rt);
                fr_canon_to_bytes(fs.rc, a.point_out + 32ull * t);
                rt_sm = rt;
            }
        }
        __syncthreads();
        const fr_t rt = rt_sm;
        fr_t nv[2];
        int cnt = 0;
        for (int e = tid; e < 8 * np; e += blockDim.x) {
            int k = e / np, b = e % np;
            nv[cnt++] = fr_add(T[k][2 * b], fr_mul_cold(rt, fr_sub(T[k][2 * b + 1], T[k][2 * b])));
        }
        __syncthreads();
        cnt = 0;
        for (int e = tid; e < 8 * np; e += blockDim.x) T[e / np][e % np] = nv[cnt++];
        __syncthreads();
    }
    if (tid < 32) {
        fr_t fin = tid == 0 ? T[0][0] : tid == 1 ? T[1][0] : fr_sub(fr_one(), T[2][0]);
        fs_absorb_frs(fs, "relu/final", fin, 3, a.finals_out);
        fs_end(fs, a.st);
    }
}

// ---------------------------------------------------------------- driver
__global__ void k_canon_to_mont(const uint8_t* in, uint32_t n, fr_t* out);   // n1.cu

void relu_prove_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* Z, const int32_t* GA, uint32_t logD, uint32_t Q,
                    uint32_t R, ReluOutputs& out, unsigned int* range_flag, Scratch& s, const uint8_t* d_pts) {
    const uint32_t QR = Q + R;
    const uint32_t logB = relu_logB(Q, R), B = 1u << logB;
    const uint64_t D = 1ull << logD;
    const uint32_t qr_mask = QR >= 32 ? 0xffffffffu : ((1u << QR) - 1);
    const uint32_t m = logB + logD;
    uint8_t* proof = out.d_proof;
    if (QR < 32) ZK_LAUNCH(ctx, k_relu_range, grid_for(ctx, D, 256, 8), 256, 0, Z, GA, D, QR, range_flag);
    // header
    uint8_t hdr[12];
    const uint32_t hv[3] = {logD, Q, R};
    for (int i = 0; i < 3; i++)
        for (int k = 0; k < 4; k++) hdr[4 * i + k] = (uint8_t)(hv[i] >> (8 * k));
    tr_absorb_host(tr, "relu/hdr", hdr, 12, proof);
    // points u_Z, u_A, u_GA, u_GZ
    fr_t* U = s.alloc<fr_t>(4ull * logD);
    if (d_pts) {   // chained (D25): the window's merged claims give the points; nothing is drawn
        ZK_LAUNCH(ctx, k_canon_to_mont, 1, 128, 0, d_pts, 4 * logD, U);
    } else {
        const char* tags[4] = {"relu/uZ", "relu/uA", "relu/uGA", "relu/uGZ"};
        const uint32_t ns[4] = {logD, logD, logD, logD};
        fr_t* outs[4] = {U, U + logD, U + 2 * logD, U + 3 * logD};
        tr_challenges_multi_dev(tr, 4, tags, ns, outs);
    }
    // claims Z~(u_Z), A~(u_A), G_A~(u_GA), G_Z~(u_GZ) with A, G_Z formed on the fly (Lemma 1)
    fr_t* claims = s.alloc<fr_t>(4);
    mle_i32_relu4(ctx, Z, GA, R, logD, U, claims, s);
    ZK_LAUNCH(ctx, k_tr_absorb_frs, 1, 32, 0, tr->d_st, make_tag("relu/claims"), (const fr_t*)claims, 4u, proof + 12);
    // r, r', u_bin
    fr_t* rr = s.alloc<fr_t>(2);
    fr_t* ubin = s.alloc<fr_t>(m);
    {
        const char* tags[3] = {"relu/r", "relu/rp", "relu/ubin"};
        const uint32_t ns[3] = {1, 1, m};
        fr_t* outs[3] = {rr, rr + 1, ubin};
        tr_challenges_multi_dev(tr, 3, tags, ns, outs);
    }
    const fr_t* u_i[5] = {U, U + logD, U + 2 * logD, U + 3 * logD, ubin + logB};

    // ---- bit sums
    // cells (cell_decode): 4B linear cells, then two upper triangles of co-occurrence cells
    const uint32_t ncell = 4 * B + B * (B + 1);
    fr_t* cell_tot = s.alloc<fr_t>(ncell);
    static const bool no_gram = getenv("ZKDL_NO_GRAM") != nullptr;   // A/B switch for the CUDA-core path
    const bool gram = relu_gram_supported(logD, B) && !no_gram;
    fr_t* lin6 = gram ? s.alloc<fr_t>(12ull * B) : nullptr;
    if (gram) {
        relu_bitsums_gram(ctx, Z, GA, logD, qr_mask, QR - 1, B, u_i, cell_tot, lin6, s);
    } else {
    const uint32_t lo_bits = logD < 12 ? logD : 12, hi_bits = logD - lo_bits;
    BitsumArgs ba;
    memset(&ba, 0, sizeof ba);
    ba.Z = Z;
    ba.GA = GA;
    ba.logD = logD;
    ba.lo_bits = lo_bits;
    ba.qr_mask = qr_mask;
    ba.sig_bit = QR - 1;
    for (int x = 0; x < 5; x++) {
        fr_t* lo = s.alloc<fr_t>(1ull << lo_bits);
        fr_t* hi = s.alloc<fr_t>(1ull << hi_bits);
        eq_table_r2_dev(ctx, u_i[x], lo_bits, lo, s);
        eq_table_dev(ctx, u_i[x] + lo_bits, hi_bits, nullptr, hi, s);
        ba.LO[x] = lo;
        ba.HI[x] = hi;
    }
    ba.B = B;
    ba.ncell = ncell;
    if (logD >= 6) {   // subset-sum tables over chunks of 64 entries
        ZK_REQUIRE(ncell <= BS2_MAXC * BS2_T, ZK_ERR_INTERNAL, "bitsum cells");
        Bitsum2Args b2;
        memset(&b2, 0, sizeof b2);
        b2.Z = Z;
        b2.GA = GA;
        b2.logD = logD;
        b2.lo_bits = lo_bits;
        b2.qr_mask = qr_mask;
        b2.sig_bit = QR - 1;
        for (int x = 0; x < 5; x++) {
            b2.LO[x] = ba.LO[x];
            b2.HI[x] = ba.HI[x];
        }
        b2.B = B;
        b2.nM = 4 * B;
        b2.nC = ncell - 4 * B;
        const uint64_t nchunks = D / BS2_CH;
        const uint32_t grid = (uint32_t)(nchunks < (uint64_t)ctx->num_sms ? nchunks : (uint64_t)ctx->num_sms);
        b2.partials = s.alloc_zero<fr_t>((size_t)grid * ncell);
        const size_t smem = sizeof(Bitsum2Smem);
        ZK_CUDA(cudaFuncSetAttribute(k_relu_bitsums2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        ZK_LAUNCH(ctx, k_relu_bitsums2, grid, BS2_T, smem, b2);
        ZK_LAUNCH(ctx, k_relu_bitsums_reduce, (ncell + 127) / 128, 128, 0, (const fr_t*)b2.partials, grid, ncell, cell_tot);
    } else {           // tiny D: one masked lazy addition per (entry, cell)
        uint32_t bs_threads = ((ncell + 1) / 2 + 31) / 32 * 32;
        if (bs_threads > 640) bs_threads = 640;
        uint64_t nchunks = D / (D < BS_CH ? D : BS_CH);
        uint32_t bs_grid = (uint32_t)(nchunks < (uint64_t)ctx->num_sms * 2 ? nchunks : (uint64_t)ctx->num_sms * 2);
        ba.partials = s.alloc<fr_t>((size_t)bs_grid * ncell);
        size_t bs_smem = 5 * BS_CH * sizeof(fr_t) + 2 * BS_CH * 4 + BS_CH;
        ZK_CUDA(cudaFuncSetAttribute(k_relu_bitsums, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bs_smem));
        ZK_REQUIRE(ncell <= 2 * bs_threads, ZK_ERR_INTERNAL, "bitsum cells exceed the block");
        ZK_LAUNCH(ctx, k_relu_bitsums, bs_grid, bs_threads, bs_smem, ba);
        ZK_LAUNCH(ctx, k_relu_bitsums_reduce, (ncell + 127) / 128, 128, 0, (const fr_t*)ba.partials, bs_grid, ncell,
                  cell_tot);
    }
    }

    // ---- j-rounds
    const uint32_t nbytes = (B + 7) / 8;
    fr_t* byte_tab = s.alloc<fr_t>(256ull * nbytes);
    fr_t* kappa = s.alloc<fr_t>(8);
    fr_t* r_all = s.alloc<fr_t>(m);
    JRoundArgs ja;
    memset(&ja, 0, sizeof ja);
    ja.cells = cell_tot;
    ja.B = B;
    ja.logB = logB;
    ja.Q = Q;
    ja.R = R;
    ja.r = rr;
    ja.ubin = ubin;
    ja.st = tr->d_st;
    ja.msg_out = proof + 140;
    ja.point_out = out.d_point;
    ja.rj_out = r_all;
    ja.byte_tab = byte_tab;
    ja.kappa = kappa;
    // derived X = 1 in the factored i-rounds (ZKDL_IR_DERIVE=0: every total from the pairs)
    static const bool derive_off = getenv("ZKDL_IR_DERIVE") && atoi(getenv("ZKDL_IR_DERIVE")) == 0;
    const bool unfactored_ = getenv("ZKDL_IROUND_V") && atoi(getenv("ZKDL_IROUND_V")) == 0;
    const bool derive = !derive_off && !unfactored_;
    fr_t* sigma = derive ? s.alloc<fr_t>(5) : nullptr;
    ja.sigma = sigma;
    // the first i-round's linear terms from the bit-sum cells (gram.cu lin6; ZKDL_IR_CELLS=0: from the pairs);
    // needs the word-sourced derived round 0 (decided below: t0 >= 2, the factored kernel)
    static const bool cells_off = getenv("ZKDL_IR_CELLS") && atoi(getenv("ZKDL_IR_CELLS")) == 0;
    fr_t* r0ext = nullptr;
    fr_t* uinv = nullptr;
    if (derive) {   // u_x[t]^-1 for every i-round (Fermat, ~0.2 ms) on the aux stream, behind the bit sums
        uinv = s.alloc<fr_t>(5ull * logD);
        UPts P;
        for (int x = 0; x < 5; x++) P.u[x] = u_i[x];
        cudaStream_t aux = ctx->aux_stream();
        ZK_CUDA(cudaEventRecord(ctx->aux_ev[0], ctx->stream));
        ZK_CUDA(cudaStreamWaitEvent(aux, ctx->aux_ev[0], 0));
        k_relu_uinv<<<(5 * logD + 3) / 4, 128, 0, aux>>>(P, logD, uinv);
        after_launch(ctx, "k_relu_uinv");
    }
    // the i-phase LO tables (eq over the first H i-variables; no kappa) on the aux stream too, beside the j-rounds
    const uint32_t hb = logD < 5 ? logD : 5;
    const uint32_t H = logD - hb;
    fr_t* LOs[5][2];
    {
        EqJob lj[5];
        uint32_t nl = 0;
        for (int x = 0; x < 5; x++) {
            LOs[x][0] = LOs[x][1] = nullptr;
            if (H) {
                LOs[x][0] = s.alloc<fr_t>(1ull << H);
                LOs[x][1] = s.alloc<fr_t>(1ull << (H - 1));
                lj[nl++] = EqJob{u_i[x], H, nullptr, 0, LOs[x][0]};
            }
        }
        if (nl) {
            cudaStream_t aux = ctx->aux_stream();
            if (!derive) {   // (the u^-1 kernel forked the aux stream otherwise)
                ZK_CUDA(cudaEventRecord(ctx->aux_ev[0], ctx->stream));
                ZK_CUDA(cudaStreamWaitEvent(aux, ctx->aux_ev[0], 0));
            }
            cudaStream_t main_stream = ctx->stream;
            ctx->stream = aux;   // eq_tables_batch launches on the context stream
            try {
                eq_tables_batch(ctx, nl, lj, s);
            } catch (...) {
                ctx->stream = main_stream;
                throw;
            }
            ctx->stream = main_stream;
        }
    }
    const bool aux_used = derive || H > 0;
    if (aux_used) ZK_CUDA(cudaEventRecord(ctx->aux_ev[1], ctx->aux_stream()));
    {   // t0 >= 2 and the factored kernel (the word-sourced rounds 0 / 1), as decided below
        const uint32_t hb_ = logD < 5 ? logD : 5, H_ = logD - hb_;
        const int plog_ = getenv("ZKDL_IPERSIST_LOG") ? atoi(getenv("ZKDL_IPERSIST_LOG")) : 16;
        const bool unf_ = getenv("ZKDL_IROUND_V") && atoi(getenv("ZKDL_IROUND_V")) == 0;
        const bool words_off_ = getenv("ZKDL_RELU_WORDS") && atoi(getenv("ZKDL_RELU_WORDS")) == 0;
        uint32_t t0_ = H_;
        if (!unf_ && ((ctx->num_sms - 1) >> hb_) >= 1 && plog_ >= 0)
            for (uint32_t t = 1; t < H_; t++)
                if ((D >> (t + 1)) <= (1ull << plog_)) {
                    t0_ = t;
                    break;
                }
        if (gram && derive && !cells_off && !unf_ && t0_ >= 2 && !words_off_) {
            r0ext = s.alloc<fr_t>(6);
            ja.r0cells = lin6;
            ja.r0ext = r0ext;
        }
    }
    ZK_LAUNCH(ctx, k_relu_jrounds, 1, 256, 0, ja);

    fr_t* HIs[6];
    EqJob jobs[11];
    uint32_t nj = 0;
    for (int x = 0; x < 5; x++) {   // (the LO tables were built on the aux stream beside the j-rounds)
        HIs[x] = s.alloc<fr_t>(1ull << hb);
        jobs[nj++] = EqJob{u_i[x] + H, hb, kappa + (x < 4 ? x : 4), 0, HIs[x]};
        if (x == 4) {   // E_b' = r' E_b for the a1 side of the AIVP
            HIs[5] = s.alloc<fr_t>(1ull << hb);
            jobs[nj++] = EqJob{u_i[4] + H, hb, kappa + 7, 0, HIs[5]};
        }
    }
    eq_tables_batch(ctx, nj, jobs, s);   // the HI tables (they need kappa from the j-rounds)
    fr_t* buf[2][3];
    for (int k = 0; k < 3; k++) {
        buf[1][k] = s.alloc<fr_t>(D >> 1);
        buf[0][k] = s.alloc<fr_t>(D >= 4 ? D >> 2 : 1);
    }
    unsigned int max_grid = (unsigned int)ctx->num_sms * 4;   // >= the factored kernel's grid (cap above)
    fr_t* partials = s.alloc<fr_t>((size_t)max_grid * 13);
    unsigned int* ticket = s.alloc_zero<unsigned int>(1);
    int lo_level = 0;
    // A/B switches (read per call, so tests can cover every path in one process): ZKDL_IROUND_V=0 the
    // unfactored round kernel; rounds with at most 2^ZKDL_IPERSIST_LOG pairs (default 16, < 0: none) run
    // in one persistent launch (k_relu_ipersist)
    const bool unfactored = getenv("ZKDL_IROUND_V") && atoi(getenv("ZKDL_IROUND_V")) == 0;
    const int plog = getenv("ZKDL_IPERSIST_LOG") ? atoi(getenv("ZKDL_IPERSIST_LOG")) : 16;
    const uint32_t pcpb = (uint32_t)((ctx->num_sms - 1) >> hb);
    uint32_t t0 = H;
    if (!unfactored && pcpb >= 1 && plog >= 0)
        for (uint32_t t = 1; t < H; t++)
            if ((D >> (t + 1)) <= (1ull << plog)) {
                t0 = t;
                break;
            }
    // ---- i-phase tables: rounds 0 and 1 of the factored kernel read the int32 words through the byte table
    // (MODE 2 / 3 of k_relu_iround_f); the Fr tables a0, a1, oms are materialised only for the other paths
    // (ZKDL_RELU_WORDS=0 forces them)
    static const bool words_off = getenv("ZKDL_RELU_WORDS") && atoi(getenv("ZKDL_RELU_WORDS")) == 0;
    const bool words = !unfactored && t0 >= 2 && !words_off;
    fr_t* full[3] = {nullptr, nullptr, nullptr};
    if (!words) {
        for (int k = 0; k < 3; k++) full[k] = s.alloc<fr_t>(D);
        ZK_LAUNCH(ctx, k_relu_materialize, grid_for(ctx, D, 256, 8), 256, 0, Z, GA, D, qr_mask, QR - 1, nbytes,
                  (const fr_t*)byte_tab, full[0], full[1], full[2]);
    }
    const fr_t* cur[3] = {full[0], full[1], full[2]};
    const size_t tb_smem = 2ull * nbytes * 256 * sizeof(fr_t);
    if (words) {
        ZK_CUDA(cudaFuncSetAttribute(k_relu_iround_f<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tb_smem));
        ZK_CUDA(cudaFuncSetAttribute(k_relu_iround_f<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tb_smem));
        ZK_CUDA(cudaFuncSetAttribute(k_relu_iround_f<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tb_smem));
        ZK_CUDA(cudaFuncSetAttribute(k_relu_iround_f<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tb_smem));
        ZK_CUDA(cudaFuncSetAttribute(k_relu_iround_f<14>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tb_smem));
    }
    ZK_REQUIRE(!r0ext || words, ZK_ERR_INTERNAL, "cell-sourced round 0 without the word-sourced rounds");
    if (aux_used) ZK_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->aux_ev[1], 0));   // u^-1, LO tables before round 0
    for (uint32_t t = 0; t < t0; t++) {
        IRoundArgs a;
        memset(&a, 0, sizeof a);
        const bool fold = t > 0;
        for (int k = 0; k < 3; k++) {
            a.src[k] = cur[k];
            a.dst[k] = fold ? buf[t & 1][k] : nullptr;
        }
        a.n_pairs = D >> (t + 1);
        a.r_prev = fold ? r_all + logB + t - 1 : nullptr;
        for (int x = 0; x < 5; x++) {
            a.lo_cur[x] = LOs[x][lo_level];
            a.lo_next[x] = LOs[x][lo_level ^ 1];
            a.hi[x] = HIs[x];
            a.u[x] = u_i[x];
        }
        a.hi[5] = HIs[5];
        a.lo_cnt = H - t;
        a.hb = hb;
        a.t = t;
        a.claim = kappa + 6;
        a.partials = partials;
        a.ticket = ticket;
        a.st = tr->d_st;
        a.msg_out = proof + 140 + 128ull * (logB + t);
        a.r_out = r_all + logB + t;
        a.point_out = out.d_point + 32ull * (logB + t);
        a.sigma = sigma;
        a.uinv = derive ? uinv + 5ull * t : nullptr;
        a.r0ext = r0ext;
        if (unfactored) {
            const unsigned int grid = grid_for(ctx, 2 * a.n_pairs, 256, 2);   // two threads per pair
            if (fold)
                ZK_LAUNCH(ctx, k_relu_iround<true>, grid, 256, 0, a);
            else
                ZK_LAUNCH(ctx, k_relu_iround<false>, grid, 256, 0, a);
        } else {
            // grid = 2^hb HI blocks x cpb CTAs each, two 256-thread CTAs per SM (ZKDL_IROUND_T=128: four
            // 128-thread CTAs; measured no better in the C4 window)
            const uint32_t ithreads = ZKDL_IR_LB_T;
            const uint64_t per_blk = a.n_pairs >> hb;
            uint64_t cpb = (per_blk + ithreads / 2 - 1) / (ithreads / 2);
            const uint64_t cap = ((uint64_t)ctx->num_sms * ZKDL_IR_LB_B) >> hb;
            if (cpb > cap) cpb = cap;
            if (cpb < 1) cpb = 1;
            a.cpb = (uint32_t)cpb;
            const unsigned int grid = (unsigned int)(cpb << hb);
            if (words && t <= 1) {
                a.words[0] = Z;
                a.words[1] = GA;
                a.byte_tab = byte_tab;
                a.qr_mask = qr_mask;
                a.sig_bit = QR - 1;
                a.nbytes = nbytes;
                if (fold && derive)
                    ZK_LAUNCH(ctx, k_relu_iround_f<7>, grid, ithreads, tb_smem, a);
                else if (fold)
                    ZK_LAUNCH(ctx, k_relu_iround_f<3>, grid, ithreads, tb_smem, a);
                else if (derive && r0ext)
                    ZK_LAUNCH(ctx, k_relu_iround_f<14>, grid, ithreads, tb_smem / 2, a);
                else if (derive)
                    ZK_LAUNCH(ctx, k_relu_iround_f<6>, grid, ithreads, tb_smem / 2, a);
                else
                    ZK_LAUNCH(ctx, k_relu_iround_f<2>, grid, ithreads, tb_smem / 2, a);
            } else if (fold) {
                if (derive)
                    ZK_LAUNCH(ctx, k_relu_iround_f<5>, grid, ithreads, 0, a);
                else
                    ZK_LAUNCH(ctx, k_relu_iround_f<1>, grid, ithreads, 0, a);
            } else {
                if (derive)
                    ZK_LAUNCH(ctx, k_relu_iround_f<4>, grid, ithreads, 0, a);
                else
                    ZK_LAUNCH(ctx, k_relu_iround_f<0>, grid, ithreads, 0, a);
            }
        }
        lo_level ^= 1;
        if (fold)
            for (int k = 0; k < 3; k++) cur[k] = buf[t & 1][k];
    }
    if (t0 < H) {
        IPersistArgs pa;
        memset(&pa, 0, sizeof pa);
        for (int k = 0; k < 3; k++) {
            pa.full[k] = full[k];
            pa.buf[0][k] = buf[0][k];
            pa.buf[1][k] = buf[1][k];
        }
        for (int x = 0; x < 5; x++) {
            pa.LO[x][0] = LOs[x][0];
            pa.LO[x][1] = LOs[x][1];
            pa.u[x] = u_i[x];
        }
        for (int x = 0; x < 6; x++) {
            pa.hi[0][x] = HIs[x];
            pa.hi[1][x] = s.alloc<fr_t>(1ull << hb);
        }
        pa.t0 = t0;
        pa.t1 = H;
        pa.H = H;
        pa.hb = hb;
        pa.cpb = pcpb;
        pa.claim = kappa + 6;
        pa.r_i = r_all + logB;
        pa.msg_base = proof + 140 + 128ull * logB;
        pa.point_base = out.d_point + 32ull * logB;
        pa.st = tr->d_st;
        const unsigned int grid = 1 + (pcpb << hb);
        pa.partials = s.alloc<fr_t>((size_t)grid * IR_NV);
        pa.sigma = sigma;
        pa.uinv = uinv;
        unsigned int* ctr = s.alloc_zero<unsigned int>(3);
        pa.arrive = ctr;
        pa.flag = ctr + 1;
        pa.hiflag = ctr + 2;
        static const bool trace = getenv("ZKDL_IPERSIST_TRACE") != nullptr;
        if (trace) pa.trace = s.alloc_zero<unsigned long long>(8ull * (H - t0) + 1);
        void* args[] = {(void*)&pa};
        cudaEvent_t ev_a = nullptr, ev_b = nullptr;
        const bool prof = ctx->prof_match("k_relu_ipersist");
        if (prof) {
            ev_a = ctx->take_event();
            ev_b = ctx->take_event();
            cudaEventRecord(ev_a, ctx->stream);
        }
        if (derive)
            ZK_CUDA(cudaLaunchCooperativeKernel((const void*)k_relu_ipersist<true>, dim3(grid), dim3(256), args, 0, ctx->stream));
        else
            ZK_CUDA(cudaLaunchCooperativeKernel((const void*)k_relu_ipersist<false>, dim3(grid), dim3(256), args, 0, ctx->stream));
        after_launch(ctx, "k_relu_ipersist");
        if (prof) {
            cudaEventRecord(ev_b, ctx->stream);
            ctx->recs.push_back({"k_relu_ipersist", ev_a, ev_b});
        }
        for (int k = 0; k < 3; k++) cur[k] = buf[(H - 1) & 1][k];
        if ((H - t0) & 1)   // the last persistent round rescaled HI' into the second buffer
            for (int x = 0; x < 6; x++) HIs[x] = pa.hi[1][x];
        if (trace) {
            std::vector<unsigned long long> h(8ull * (H - t0));
            ZK_CUDA(cudaMemcpyAsync(h.data(), pa.trace, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
            ZK_CUDA(cudaStreamSynchronize(ctx->stream));
            for (uint32_t t = t0; t < H; t++) {
                const unsigned long long* q = &h[4ull * (t - t0)];
                const unsigned long long prev = t > t0 ? h[4ull * (t - t0) - 2] : q[0];
                const unsigned long long* wq = &h[4ull * (H - t0) + 4ull * (t - t0)];
                fprintf(stderr, "ipersist t=%u workers %.1f us, reduce %.1f, g+transcript %.1f, update %.1f | worker1: "
                        "woke +%.1f, pairs %.1f, hi wait %.1f, reduce+publish %.1f\n", t,
                        (q[0] - prev) / 1e3, (q[1] - q[0]) / 1e3, (q[2] - q[1]) / 1e3, (q[3] - q[2]) / 1e3,
                        ((long long)wq[0] - (long long)prev) / 1e3, (wq[1] - wq[0]) / 1e3, (wq[2] - wq[1]) / 1e3,
                        (wq[3] - wq[2]) / 1e3);
            }
        }
    }
    ITailArgs ta;
    memset(&ta, 0, sizeof ta);
    for (int k = 0; k < 3; k++) ta.src[k] = cur[k];
    ta.fold = H > 0;
    ta.r_prev = H > 0 ? r_all + logB + H - 1 : nullptr;
    for (int x = 0; x < 5; x++) ta.hi[x] = HIs[x];
    ta.hb = hb;
    ta.kappa = kappa;
    ta.st = tr->d_st;
    ta.msg_out = proof + 140 + 128ull * (logB + H);
    ta.point_out = out.d_point + 32ull * (logB + H);
    ta.r_out = r_all + logB + H;
    ta.finals_out = proof + 140 + 128ull * m;
    ZK_LAUNCH(ctx, k_relu_itail, 1, 256, 0, ta);
}

}  // namespace zk
