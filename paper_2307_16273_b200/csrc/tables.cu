// tables.cu — rows a1 (embed) and a2 (eq / MLE), conversions, and the shared reductions.
#include "tables.cuh"

namespace zk {

// ---------------------------------------------------------------- a1: embed int32 -> Fr
__global__ void k_embed_i32(const int32_t* in, uint64_t n, fr_t* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        fr_store(&out[i], fr_from_i32(__ldg(in + i)));
}

void embed_i32_dev(zk_ctx* ctx, const int32_t* d_in, uint64_t n, fr_t* d_out) {
    if (!n) return;
    ZK_LAUNCH(ctx, k_embed_i32, grid_for(ctx, n, 256, 8), 256, 0, d_in, n, d_out);
}

// ---------------------------------------------------------------- conversions
__global__ void k_to_canonical(const fr_t* in, uint64_t n, fr_t* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        fr_store(&out[i], fr_to_canonical(fr_load(&in[i])));
}
__device__ __forceinline__ bool lt_p(const fr_t& x) {
    const uint32_t P_[8] = {ZK_P0, ZK_P1, ZK_P2, ZK_P3, ZK_P4, ZK_P5, ZK_P6, ZK_P7};
    for (int i = 7; i >= 0; i--) {
        if (x.v[i] < P_[i]) return true;
        if (x.v[i] > P_[i]) return false;
    }
    return false;
}
__global__ void k_from_canonical(const fr_t* in, uint64_t n, fr_t* out, unsigned int* bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        fr_t x = fr_load(&in[i]);
        if (!lt_p(x)) atomicOr(bad, 1u);
        fr_store(&out[i], fr_from_canonical(x));
    }
}

void to_canonical_dev(zk_ctx* ctx, const fr_t* in, uint64_t n, uint8_t* out) {
    if (!n) return;
    ZK_LAUNCH(ctx, k_to_canonical, grid_for(ctx, n, 256, 8), 256, 0, in, n, reinterpret_cast<fr_t*>(out));
}

// Points travel in the kernel parameters (copied at launch): no staging buffer, no stream sync.
struct Pts96 {
    uint32_t n;
    uint8_t b[96][32];
};
__global__ void k_upload_pts(Pts96 p, fr_t* out) {
    const uint32_t i = threadIdx.x;
    if (i < p.n) {
        fr_t x;
        for (int k = 0; k < 8; k++)
            x.v[k] = (uint32_t)p.b[i][4 * k] | ((uint32_t)p.b[i][4 * k + 1] << 8) | ((uint32_t)p.b[i][4 * k + 2] << 16) |
                     ((uint32_t)p.b[i][4 * k + 3] << 24);
        fr_store(&out[i], fr_from_canonical(x));
    }
}

void upload_points(zk_ctx* ctx, const zk_fr* host, uint32_t n, fr_t* d_mont, Scratch& s) {
    (void)s;
    if (!n) return;
    check_canonical(host, n);   // host-side validation (ZK_ERR_NONCANONICAL)
    for (uint32_t off = 0; off < n; off += 96) {
        Pts96 p;
        p.n = n - off < 96 ? n - off : 96;
        memcpy(p.b, host + off, 32ull * p.n);
        ZK_LAUNCH(ctx, k_upload_pts, 1, 96, 0, p, d_mont + off);
    }
}

// ---------------------------------------------------------------- a2: eq tables
// Direct product per entry: out[x] = scale * prod_{s<k} (bit_s(x) ? u_s : 1 - u_s); used for k <= 12.
__global__ void k_eq_direct(const fr_t* u, uint32_t k, const fr_t* scale, fr_t* out) {
    const uint64_t n = 1ull << k;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) {
        fr_t acc = scale ? fr_load(scale) : fr_one();
        for (uint32_t t = 0; t < k; t++) {
            fr_t ut = fr_load(&u[t]);
            acc = fr_mul(acc, ((x >> t) & 1) ? ut : fr_sub(fr_one(), ut));
        }
        fr_store(&out[x], acc);
    }
}
// out[x] = lo[x & (2^klo - 1)] * hi[x >> klo]
__global__ void k_eq_combine(const fr_t* lo, const fr_t* hi, uint32_t klo, uint64_t n, fr_t* out) {
    const uint64_t mask = (1ull << klo) - 1;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x)
        fr_store(&out[x], fr_mul(fr_load(&lo[x & mask]), fr_load(&hi[x >> klo])));
}

void eq_table_dev(zk_ctx* ctx, const fr_t* d_u, uint32_t k, const fr_t* d_scale, fr_t* d_out, Scratch& s) {
    if (k <= 10) {
        ZK_LAUNCH(ctx, k_eq_direct, grid_for(ctx, 1ull << k, 128, 8), 128, 0, d_u, k, d_scale, d_out);
        return;
    }
    uint32_t klo = (k + 1) / 2, khi = k - klo;
    fr_t* lo = s.alloc<fr_t>(1ull << klo);
    fr_t* hi = s.alloc<fr_t>(1ull << khi);
    ZK_LAUNCH(ctx, k_eq_direct, grid_for(ctx, 1ull << klo, 128, 8), 128, 0, d_u, klo, (const fr_t*)nullptr, lo);
    ZK_LAUNCH(ctx, k_eq_direct, grid_for(ctx, 1ull << khi, 128, 8), 128, 0, d_u + klo, khi, d_scale, hi);
    ZK_LAUNCH(ctx, k_eq_combine, grid_for(ctx, 1ull << k, 256, 8), 256, 0, lo, hi, klo, 1ull << k, d_out);
}

__global__ void k_set_const(fr_t* out, fr_t v) { fr_store(out, v); }

// ---------------------------------------------------------------- batched eq tables
// Phase 1: every direct table of the batch (the small tables whole, the large ones' lo and hi halves)
// in one launch; phase 2: every lo x hi combine in one launch.  Entry x of part p belongs to the part
// whose [start, start + 2^k) range contains the flat index (binary search over <= 2 EQB_MAX parts).
struct EqParts {
    uint32_t n;
    uint64_t start[2 * EQB_MAX + 1];
    const fr_t* u[2 * EQB_MAX];
    const fr_t* scale[2 * EQB_MAX];
    fr_t* out[2 * EQB_MAX];
    uint32_t k[2 * EQB_MAX];
    int r2[2 * EQB_MAX];   // scale is R (the "double Montgomery" tables of the lazy int32 dot products)
};
__global__ void k_eq_direct_batch(EqParts P) {
    const uint64_t total = P.start[P.n];
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total; g += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = P.n;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (P.start[mid] <= g) lo = mid; else hi = mid;
        }
        const uint64_t x = g - P.start[lo];
        fr_t acc = P.r2[lo] ? ZK_R2 : (P.scale[lo] ? fr_load(P.scale[lo]) : fr_one());
        for (uint32_t t = 0; t < P.k[lo]; t++) {
            const fr_t ut = fr_load(&P.u[lo][t]);
            acc = fr_mul(acc, ((x >> t) & 1) ? ut : fr_sub(fr_one(), ut));
        }
        fr_store(&P.out[lo][x], acc);
    }
}
struct EqCombines {
    uint32_t n;
    uint64_t start[EQB_MAX + 1];
    const fr_t* lo[EQB_MAX];
    const fr_t* hi[EQB_MAX];
    fr_t* out[EQB_MAX];
    uint32_t klo[EQB_MAX];
};
__global__ void k_eq_combine_batch(EqCombines C) {
    const uint64_t total = C.start[C.n];
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total; g += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = C.n;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (C.start[mid] <= g) lo = mid; else hi = mid;
        }
        const uint64_t x = g - C.start[lo];
        const uint64_t mask = (1ull << C.klo[lo]) - 1;
        fr_store(&C.out[lo][x], fr_mul(fr_load(&C.lo[lo][x & mask]), fr_load(&C.hi[lo][x >> C.klo[lo]])));
    }
}

void eq_tables_batch(zk_ctx* ctx, uint32_t n, const EqJob* jobs, Scratch& s) {
    for (uint32_t b0 = 0; b0 < n; b0 += EQB_MAX) {
        const uint32_t nb = n - b0 < EQB_MAX ? n - b0 : EQB_MAX;
        EqParts P;
        EqCombines C;
        memset(&P, 0, sizeof P);
        memset(&C, 0, sizeof C);
        for (uint32_t i = 0; i < nb; i++) {
            const EqJob& J = jobs[b0 + i];
            auto part = [&](const fr_t* u, uint32_t k, const fr_t* sc, int r2, fr_t* out) {
                P.u[P.n] = u;
                P.k[P.n] = k;
                P.scale[P.n] = sc;
                P.r2[P.n] = r2;
                P.out[P.n] = out;
                P.start[P.n + 1] = P.start[P.n] + (1ull << k);
                P.n++;
            };
            if (J.k <= 10) {
                part(J.u, J.k, J.scale, J.r2, J.out);
            } else {
                const uint32_t klo = (J.k + 1) / 2, khi = J.k - klo;
                fr_t* lo = s.alloc<fr_t>(1ull << klo);
                fr_t* hi = s.alloc<fr_t>(1ull << khi);
                part(J.u, klo, nullptr, 0, lo);
                part(J.u + klo, khi, J.scale, J.r2, hi);
                C.lo[C.n] = lo;
                C.hi[C.n] = hi;
                C.out[C.n] = J.out;
                C.klo[C.n] = klo;
                C.start[C.n + 1] = C.start[C.n] + (1ull << J.k);
                C.n++;
            }
        }
        ZK_LAUNCH(ctx, k_eq_direct_batch, grid_for(ctx, P.start[P.n], 128, 8), 128, 0, P);
        if (C.n) ZK_LAUNCH(ctx, k_eq_combine_batch, grid_for(ctx, C.start[C.n], 256, 8), 256, 0, C);
    }
}

void eq_table_r2_dev(zk_ctx* ctx, const fr_t* d_u, uint32_t k, fr_t* d_out, Scratch& s) {
    // the batch kernel's r2 start value (the Montgomery form of the field element R): no constant to upload
    const EqJob j{d_u, k, nullptr, 1, d_out};
    eq_tables_batch(ctx, 1, &j, s);
}

// ---------------------------------------------------------------- dot products and MLE
__global__ void __launch_bounds__(256) k_dot_fr(const fr_t* a, const fr_t* b, uint64_t n, fr_t* partials,
                                                unsigned int* ticket, fr_t* out) {
    fr_t acc[1] = {fr_zero()};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        acc[0] = fr_add(acc[0], fr_mul(fr_load(&a[i]), fr_load(&b[i])));
    fr_t tot[1];
    if (grid_reduce_fr<1>(acc, partials, ticket, tot)) fr_store(out, tot[0]);
}

static void dot_dev(zk_ctx* ctx, const fr_t* a, const fr_t* b, uint64_t n, fr_t* d_out, Scratch& s) {
    unsigned int g = grid_for(ctx, n, 256, 2);
    fr_t* part = s.alloc<fr_t>(g);
    unsigned int* ticket = s.alloc_zero<unsigned int>(1);
    ZK_LAUNCH(ctx, k_dot_fr, g, 256, 0, a, b, n, part, ticket, d_out);
}

// Row sums of an Fr table viewed as [2^hi][2^lo] with weights lo: out[r] = sum_c T[r][c] * w[c]
__global__ void __launch_bounds__(256) k_rowdot_fr(const fr_t* T, uint64_t nrows, uint32_t cols, const fr_t* w, fr_t* out) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = warp; r < nrows; r += nwarps) {
        fr_t acc[1] = {fr_zero()};
        for (uint32_t c = lane; c < cols; c += 32) acc[0] = fr_add(acc[0], fr_mul(fr_load(&T[r * cols + c]), fr_load(&w[c])));
        warp_reduce_fr<1>(acc);
        if (lane == 0) fr_store(&out[r], acc[0]);
    }
}

static void split_bits(uint32_t m, uint32_t& lo, uint32_t& hi) {
    lo = m < 12 ? m : 12;
    hi = m - lo;
}

template <class Load>
static void mle_i32_generic(zk_ctx* ctx, Load load, uint32_t m, const fr_t* d_u, fr_t* d_out, Scratch& s) {
    uint32_t lo, hi;
    split_bits(m, lo, hi);
    fr_t* E2 = s.alloc<fr_t>(1ull << lo);
    eq_table_r2_dev(ctx, d_u, lo, E2, s);
    uint64_t rows = 1ull << hi;
    fr_t* V = s.alloc<fr_t>(rows);
    unsigned int g = grid_for(ctx, rows * 32, 256, 8);
    ZK_LAUNCH(ctx, k_rowdot_i32<Load>, g, 256, 0, load, rows, 1u << lo, E2, V, rows, hi, (uint64_t)1);
    if (hi == 0) {
        ZK_CUDA(cudaMemcpyAsync(d_out, V, 32, cudaMemcpyDeviceToDevice, ctx->stream));
        return;
    }
    fr_t* H = s.alloc<fr_t>(rows);
    eq_table_dev(ctx, d_u + lo, hi, nullptr, H, s);
    dot_dev(ctx, V, H, rows, d_out, s);
}

void mle_i32_plain(zk_ctx* ctx, const int32_t* d_tab, uint32_t m, const fr_t* d_u, fr_t* d_out, Scratch& s) {
    mle_i32_generic(ctx, LoadPlain{d_tab}, m, d_u, d_out, s);
}
void mle_i32_relu(zk_ctx* ctx, int kind, const int32_t* d_z, const int32_t* d_g, uint32_t R, uint32_t m, const fr_t* d_u,
                  fr_t* d_out, Scratch& s) {
    if (kind == 0)
        mle_i32_generic(ctx, LoadReluA{d_z, R}, m, d_u, d_out, s);
    else if (kind == 2)
        mle_i32_generic(ctx, LoadRound{d_z, R}, m, d_u, d_out, s);
    else
        mle_i32_generic(ctx, LoadReluGZ{d_z, d_g, R}, m, d_u, d_out, s);
}

// The four zkReLU claims Z~(u_Z), A~(u_A), G_A~(u_GA), G_Z~(u_GZ) (A, G_Z formed on the fly, Lemma 1):
// the eight eq tables in one batch, then a row-dot and a dot per claim.
// The four zkReLU claims Z~(u_Z), A~(u_A), G_A~(u_GA), G_Z~(u_GZ) (D3b) in one pass over Z and G_A: the
// tables viewed as [2^hi rows][256 columns] (entry i = 256 r + c, so the low 8 point coordinates index the
// column, D2); thread c of a CTA owns column c and streams a contiguous range of rows, accumulating the
// four lazy sums sum_r H_k[r] u_k[r][c] (u = v + 2^31, H_k = eq over the high coordinates, R-scaled);
// each CTA writes the four column partials as Fr (REDC without the bias); k_mle4_finish adds the CTAs'
// partials, weights column c by E_k[c] (eq over the low coordinates) and removes the bias once:
// sum_c E_k[c] sum_r H_k[r] 2^31 = 2^31.  (The former path: four row-dot launches, one warp per row and a
// 32-byte eq load per element, ~0.24 ms at C4; this one reads each word once.)
__global__ void __launch_bounds__(256) k_mle4_rows(const int32_t* Z, const int32_t* GA, uint32_t R, uint64_t rows,
                                                   const fr_t* H0, const fr_t* H1, const fr_t* H2, const fr_t* H3,
                                                   fr_t* partials) {
    // the CTA's rows of the four row tables staged in shared memory (the loop then waits only on the words),
    // and the words of the next four rows loaded while the current ones are accumulated (memory latency was
    // the bound: ncu long_sb 68%, 0.47 TB/s)
    extern __shared__ fr_t sH[];
    const uint64_t r0 = blockIdx.x * rows / gridDim.x, r1 = (blockIdx.x + 1) * rows / gridDim.x;
    const uint32_t nr = (uint32_t)(r1 - r0);
    for (uint32_t e = threadIdx.x; e < 4 * nr; e += blockDim.x) {
        const uint32_t k = e / nr, i = e % nr;
        const fr_t* H = k == 0 ? H0 : k == 1 ? H1 : k == 2 ? H2 : H3;
        sH[k * nr + i] = fr_load(&H[r0 + i]);
    }
    __syncthreads();
    const uint32_t c = threadIdx.x;
    uint32_t acc[4][10];
#pragma unroll
    for (int k = 0; k < 4; k++)
#pragma unroll
        for (int l = 0; l < 10; l++) acc[k][l] = 0;
    const int64_t half = 1ll << (R - 1);
    uint64_t r = r0;
    int32_t zn[4], gn[4];
    if (r + 3 < r1) {
#pragma unroll
        for (int i = 0; i < 4; i++) {
            zn[i] = __ldcs(Z + (r + i) * 256 + c);
            gn[i] = __ldcs(GA + (r + i) * 256 + c);
        }
    }
    for (; r + 3 < r1; r += 4) {
        int32_t z[4], g[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            z[i] = zn[i];
            g[i] = gn[i];
        }
        if (r + 7 < r1) {   // the next four rows in flight
#pragma unroll
            for (int i = 0; i < 4; i++) {
                zn[i] = __ldcs(Z + (r + 4 + i) * 256 + c);
                gn[i] = __ldcs(GA + (r + 4 + i) * 256 + c);
            }
        }
        const uint32_t o = (uint32_t)(r - r0);
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int32_t a = z[i] >= 0 ? (int32_t)(((int64_t)z[i] + half) >> R) : 0;      // A = 1{Z >= 0} round(Z / 2^R)
            const int32_t gz = z[i] >= 0 ? (int32_t)(((int64_t)g[i] + half) >> R) : 0;     // G_Z = 1{Z >= 0} round(G_A / 2^R)
            ZK_MAC_WIDE(acc[0], sH[o + i], (uint32_t)z[i] + 0x80000000u);
            ZK_MAC_WIDE(acc[1], sH[nr + o + i], (uint32_t)a + 0x80000000u);
            ZK_MAC_WIDE(acc[2], sH[2 * nr + o + i], (uint32_t)g[i] + 0x80000000u);
            ZK_MAC_WIDE(acc[3], sH[3 * nr + o + i], (uint32_t)gz + 0x80000000u);
        }
    }
    for (; r < r1; r++) {
        const int32_t z = __ldcs(Z + r * 256 + c), g = __ldcs(GA + r * 256 + c);
        const int32_t a = z >= 0 ? (int32_t)(((int64_t)z + half) >> R) : 0;
        const int32_t gz = z >= 0 ? (int32_t)(((int64_t)g + half) >> R) : 0;
        const uint32_t o = (uint32_t)(r - r0);
        ZK_MAC_WIDE(acc[0], sH[o], (uint32_t)z + 0x80000000u);
        ZK_MAC_WIDE(acc[1], sH[nr + o], (uint32_t)a + 0x80000000u);
        ZK_MAC_WIDE(acc[2], sH[2 * nr + o], (uint32_t)g + 0x80000000u);
        ZK_MAC_WIDE(acc[3], sH[3 * nr + o], (uint32_t)gz + 0x80000000u);
    }
#pragma unroll
    for (int k = 0; k < 4; k++) fr_store(&partials[((uint64_t)blockIdx.x * 4 + k) * 256 + c], fr_redc_wide(acc[k]));
}
// block (k, q, part): claim k, columns 32 q .. 32 q + 31, CTAs b = part (mod MLE4_PARTS); warp w adds the partials of
// CTAs b = part + MLE4_PARTS (w + 8 i); the column sums are weighted by E_k[c] and summed into
// mid[(k * 8 + q) * MLE4_PARTS + part]
constexpr uint32_t MLE4_PARTS = 4;
__global__ void __launch_bounds__(256) k_mle4_finish(const fr_t* partials, uint32_t nb, const fr_t* E0, const fr_t* E1,
                                                     const fr_t* E2, const fr_t* E3, fr_t* mid) {
    __shared__ fr_t sm[8][32];
    const uint32_t part = blockIdx.x % MLE4_PARTS, kq = blockIdx.x / MLE4_PARTS;
    const uint32_t k = kq >> 3, q = kq & 7, w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const uint32_t c = q * 32 + l;
    fr_t s = fr_zero();
    for (uint32_t b = part + MLE4_PARTS * w; b < nb; b += 8 * MLE4_PARTS)
        s = fr_add(s, fr_load(&partials[((uint64_t)b * 4 + k) * 256 + c]));
    sm[w][l] = s;
    __syncthreads();
    if (w == 0) {
#pragma unroll
        for (int i = 1; i < 8; i++) s = fr_add(s, sm[i][l]);
        const fr_t* E = k == 0 ? E0 : k == 1 ? E1 : k == 2 ? E2 : E3;
        fr_t v[1] = {fr_mul(s, fr_load(&E[c]))};
        warp_reduce_fr<1>(v);
        if (l == 0) fr_store(&mid[kq * MLE4_PARTS + part], v[0]);
    }
}
// out[k] = sum of mid[k * 8 * MLE4_PARTS ..] - 2^31 (the bias of the lazy sums)
__global__ void k_mle4_final(const fr_t* mid, fr_t* out) {
    const uint32_t k = threadIdx.x;
    if (k >= 4) return;
    fr_t s = fr_zero();
    for (uint32_t q = 0; q < 8 * MLE4_PARTS; q++) s = fr_add(s, fr_load(&mid[k * 8 * MLE4_PARTS + q]));
    fr_store(&out[k], fr_sub(s, ZK_TWO31_MONT));
}

void mle_i32_relu4(zk_ctx* ctx, const int32_t* d_z, const int32_t* d_g, uint32_t R, uint32_t m, const fr_t* d_U,
                   fr_t* d_out, Scratch& s) {
    static const bool fused_off = getenv("ZKDL_MLE4_FUSED") && atoi(getenv("ZKDL_MLE4_FUSED")) == 0;
    // (the fused kernel stages a CTA's rows of the four row tables in shared memory: <= 2^26 entries)
    if (!fused_off && m >= 16 && m <= 26 && R >= 1) {
        const uint32_t lo = 8, hi = m - 8;
        fr_t* E[4];
        fr_t* H[4];
        EqJob jobs[8];
        for (int c = 0; c < 4; c++) {
            E[c] = s.alloc<fr_t>(256);
            H[c] = s.alloc<fr_t>(1ull << hi);
            jobs[2 * c] = EqJob{d_U + (uint64_t)c * m, lo, nullptr, 0, E[c]};
            jobs[2 * c + 1] = EqJob{d_U + (uint64_t)c * m + lo, hi, nullptr, 1, H[c]};   // R-scaled: lazy MACs
        }
        eq_tables_batch(ctx, 8, jobs, s);
        const uint64_t rows = 1ull << hi;
        uint32_t nb = (uint32_t)ctx->num_sms * 2;
        if ((uint64_t)nb > rows / 4) nb = (uint32_t)(rows / 4);
        fr_t* P = s.alloc<fr_t>((uint64_t)nb * 4 * 256);
        const size_t hsm = 4 * sizeof(fr_t) * (size_t)((rows + nb - 1) / nb + 1);
        if (hsm > 48 * 1024)
            ZK_CUDA(cudaFuncSetAttribute(k_mle4_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm));
        ZK_LAUNCH(ctx, k_mle4_rows, nb, 256, hsm, d_z, d_g, R, rows, (const fr_t*)H[0], (const fr_t*)H[1],
                  (const fr_t*)H[2], (const fr_t*)H[3], P);
        fr_t* mid = s.alloc<fr_t>(32 * MLE4_PARTS);
        ZK_LAUNCH(ctx, k_mle4_finish, 32 * MLE4_PARTS, 256, 0, (const fr_t*)P, nb, (const fr_t*)E[0], (const fr_t*)E[1],
                  (const fr_t*)E[2], (const fr_t*)E[3], mid);
        ZK_LAUNCH(ctx, k_mle4_final, 1, 32, 0, (const fr_t*)mid, d_out);
        return;
    }
    uint32_t lo, hi;
    split_bits(m, lo, hi);
    fr_t* E2[4];
    fr_t* H[4];
    EqJob jobs[8];
    uint32_t nj = 0;
    for (int c = 0; c < 4; c++) {
        E2[c] = s.alloc<fr_t>(1ull << lo);
        jobs[nj++] = EqJob{d_U + (uint64_t)c * m, lo, nullptr, 1, E2[c]};
        H[c] = nullptr;
        if (hi) {
            H[c] = s.alloc<fr_t>(1ull << hi);
            jobs[nj++] = EqJob{d_U + (uint64_t)c * m + lo, hi, nullptr, 0, H[c]};
        }
    }
    eq_tables_batch(ctx, nj, jobs, s);
    const uint64_t rows = 1ull << hi;
    const unsigned int g = grid_for(ctx, rows * 32, 256, 8);
    for (int c = 0; c < 4; c++) {
        fr_t* V = hi ? s.alloc<fr_t>(rows) : d_out + c;
        if (c == 0) ZK_LAUNCH(ctx, k_rowdot_i32<LoadPlain>, g, 256, 0, LoadPlain{d_z}, rows, 1u << lo, (const fr_t*)E2[c], V, rows, hi, (uint64_t)1);
        if (c == 1) ZK_LAUNCH(ctx, k_rowdot_i32<LoadReluA>, g, 256, 0, LoadReluA{d_z, R}, rows, 1u << lo, (const fr_t*)E2[c], V, rows, hi, (uint64_t)1);
        if (c == 2) ZK_LAUNCH(ctx, k_rowdot_i32<LoadPlain>, g, 256, 0, LoadPlain{d_g}, rows, 1u << lo, (const fr_t*)E2[c], V, rows, hi, (uint64_t)1);
        if (c == 3) ZK_LAUNCH(ctx, k_rowdot_i32<LoadReluGZ>, g, 256, 0, LoadReluGZ{d_z, d_g, R}, rows, 1u << lo, (const fr_t*)E2[c], V, rows, hi, (uint64_t)1);
        if (hi) dot_dev(ctx, V, H[c], rows, d_out + c, s);
    }
}

void mle_fr_dev(zk_ctx* ctx, const fr_t* d_tab, uint32_t m, const fr_t* d_u, fr_t* d_out, Scratch& s) {
    uint32_t lo, hi;
    split_bits(m, lo, hi);
    fr_t* E = s.alloc<fr_t>(1ull << lo);
    eq_table_dev(ctx, d_u, lo, nullptr, E, s);
    uint64_t rows = 1ull << hi;
    fr_t* V = s.alloc<fr_t>(rows);
    ZK_LAUNCH(ctx, k_rowdot_fr, grid_for(ctx, rows * 32, 256, 8), 256, 0, d_tab, rows, 1u << lo, E, V);
    if (hi == 0) {
        ZK_CUDA(cudaMemcpyAsync(d_out, V, 32, cudaMemcpyDeviceToDevice, ctx->stream));
        return;
    }
    fr_t* H = s.alloc<fr_t>(rows);
    eq_table_dev(ctx, d_u + lo, hi, nullptr, H, s);
    dot_dev(ctx, V, H, rows, d_out, s);
}

// ---------------------------------------------------------------- diagnostics: element-wise field ops
__global__ void k_selftest_op(int op, const fr_t* a, const fr_t* b, uint64_t n, fr_t* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        fr_t x = fr_load(&a[i]), y = b ? fr_load(&b[i]) : fr_zero(), r;
        switch (op) {
            case 0: r = fr_add(x, y); break;
            case 1: r = fr_sub(x, y); break;
            case 2: r = fr_mul(x, y); break;
            case 3: r = fr_inv(x); break;
            case 4: r = fr_neg(x); break;
            case 5: r = fr_sqr(x); break;
            case 6: r = fr_inv_bgcd(x); break;
            default: r = fr_zero();
        }
        fr_store(&out[i], r);
    }
}
void selftest_op_dev(zk_ctx* ctx, int op, const fr_t* a, const fr_t* b, uint64_t n, fr_t* out) {
    ZK_LAUNCH(ctx, k_selftest_op, grid_for(ctx, n, 128, 8), 128, 0, op, a, b, n, out);
}

// Microbenchmark: `iters` dependent-chain Montgomery products per thread on register-resident values,
// 4 independent chains per thread (measures the sustained Fr-mul throughput of this implementation).
__global__ void __launch_bounds__(256) k_mul_bench(const fr_t* seed, uint32_t iters, fr_t* out) {
    uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    fr_t a = fr_load(&seed[tid & 1023]), b = fr_load(&seed[(tid + 1) & 1023]);
    fr_t c = fr_load(&seed[(tid + 2) & 1023]), d = fr_load(&seed[(tid + 3) & 1023]);
    fr_t k = fr_load(&seed[(tid + 7) & 1023]);
    for (uint32_t i = 0; i < iters; i++) {
        a = fr_mul(a, k);
        b = fr_mul(b, k);
        c = fr_mul(c, k);
        d = fr_mul(d, k);
    }
    fr_store(&out[tid], fr_add(fr_add(a, b), fr_add(c, d)));
}
void mul_bench_dev(zk_ctx* ctx, const fr_t* seed, uint32_t iters, uint32_t blocks, fr_t* out) {
    ZK_LAUNCH(ctx, k_mul_bench, blocks, 256, 0, seed, iters, out);
}

__global__ void k_colsum_finish(const uint32_t* partials, uint64_t N, uint32_t cols, uint32_t S, fr_t* out) {
    const uint64_t outputs = N * cols;
    for (uint64_t o = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; o < outputs; o += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t acc[10];
#pragma unroll
        for (int k = 0; k < 10; k++) acc[k] = partials[o * 10 + k];
        for (uint32_t sp = 1; sp < S; sp++) {
            uint32_t b[10];
#pragma unroll
            for (int k = 0; k < 10; k++) b[k] = partials[(sp * outputs + o) * 10 + k];
            wide_add10(acc, b);
        }
        const uint64_t n = o / cols, c = o % cols;
        fr_store(&out[c * N + n], wide_finish(acc));
    }
}

// Row-streaming column sums for wide stacks (cols = 256 CS, CS in {2, 4}): the row units (n, r) of the
// whole stack are cut into one contiguous range per CTA; a CTA streams its rows whole (4 KB contiguous at
// cols = 1024; the column-strip kernel above reads 512-byte strips of 4 KB-strided rows) with thread t
// owning columns t + 256 j, and flushes one 10-limb partial per instance it touches (slot = n - first
// instance of its range); k_colsum_rows_finish adds the partials of the CTAs that cover each instance.
template <int CS>
__global__ void __launch_bounds__(256) k_colsum_rows(const int32_t* M, uint64_t N, uint32_t rows, const fr_t* E2,
                                                     uint32_t* partials, uint32_t slots) {
    constexpr uint32_t cols = 256 * CS;
    const uint64_t units = N * rows, R = gridDim.x;
    const uint64_t lo = blockIdx.x * units / R, hi = (blockIdx.x + 1) * units / R;
    const uint64_t n_first = lo / rows;
    uint64_t u = lo;
    while (u < hi) {
        const uint64_t n = u / rows, end = (n + 1) * rows < hi ? (n + 1) * rows : hi;
        uint32_t acc[CS][10];
#pragma unroll
        for (int j = 0; j < CS; j++)
#pragma unroll
            for (int k = 0; k < 10; k++) acc[j][k] = 0;
        const fr_t* Er = E2 + (u - n * rows);   // eq weight of the current row (no per-row modulo)
        const int32_t* Mr = M + u * cols + threadIdx.x;
        for (; u + 3 < end; u += 4, Er += 4, Mr += 4 * cols) {   // 4 rows x CS columns of loads in flight
            uint32_t v[4][CS];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < CS; j++) v[i][j] = (uint32_t)__ldcs(Mr + i * cols + 256 * j);
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const fr_t e = fr_load(&Er[i]);
#pragma unroll
                for (int j = 0; j < CS; j++) ZK_MAC_WIDE(acc[j], e, v[i][j] + 0x80000000u);
            }
        }
        for (; u < end; u++, Er++, Mr += cols) {
            const fr_t e = fr_load(Er);
#pragma unroll
            for (int j = 0; j < CS; j++) ZK_MAC_WIDE(acc[j], e, (uint32_t)__ldcs(Mr + 256 * j) + 0x80000000u);
        }
        uint32_t* P = partials + ((uint64_t)blockIdx.x * slots + (n - n_first)) * cols * 10;
#pragma unroll
        for (int j = 0; j < CS; j++)
#pragma unroll
            for (int k = 0; k < 10; k++) P[(uint64_t)(threadIdx.x + 256 * j) * 10 + k] = acc[j][k];
    }
}
__global__ void k_colsum_rows_finish(const uint32_t* partials, uint64_t N, uint32_t rows, uint32_t cols, uint32_t R,
                                     uint32_t slots, fr_t* out) {
    const uint64_t units = N * rows;
    for (uint64_t o = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; o < N * cols; o += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t n = o / cols, c = o % cols;
        // CTAs whose unit range [b units / R, (b + 1) units / R) meets [n rows, (n + 1) rows)
        uint64_t b = n * rows * R / units;
        while (b > 0 && b * units / R > n * rows) b--;
        while ((b + 1) * units / R <= n * rows) b++;
        uint32_t acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (; b < R && b * units / R < (n + 1) * rows; b++) {
            const uint64_t n_first = (b * units / R) / rows;
            const uint32_t* P = partials + ((b * slots + (n - n_first)) * cols + c) * 10;
            uint32_t x[10];
#pragma unroll
            for (int k = 0; k < 10; k++) x[k] = P[k];
            wide_add10(acc, x);
        }
        fr_store(&out[c * N + n], wide_finish(acc));
    }
}

void colsum_i32(zk_ctx* ctx, const int32_t* M, uint64_t N, uint32_t rows, uint32_t cols, const fr_t* E2, fr_t* out,
                Scratch& s) {
    if (colsum_tc_ok(N, rows, cols)) {   // tensor cores (TMA + MN-major int8 MMAs)
        colsum_tc(ctx, M, N, rows, cols, E2, out, s);
        return;
    }
    // wide stacks with many row units: the row-streaming kernel (ZKDL_COLSUM_ROWS=0 disables it)
    static const bool rows_off = getenv("ZKDL_COLSUM_ROWS") && atoi(getenv("ZKDL_COLSUM_ROWS")) == 0;
    if (!rows_off && (cols == 512 || cols == 1024) && N * rows >= 64ull * ctx->num_sms) {
        static int per_sm[2] = {0, 0};
        const int ci = cols == 1024;
        if (!per_sm[ci]) {
            if (ci)
                ZK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[ci], k_colsum_rows<4>, 256, 0));
            else
                ZK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[ci], k_colsum_rows<2>, 256, 0));
            if (per_sm[ci] < 1) per_sm[ci] = 1;
        }
        const uint32_t R = (uint32_t)ctx->num_sms * per_sm[ci];
        const uint64_t units = N * rows, span = (units + R - 1) / R;
        const uint32_t slots = (uint32_t)((span + rows - 1) / rows + 1);   // instances one unit range can touch
        uint32_t* partials = s.alloc<uint32_t>((uint64_t)R * slots * cols * 10);
        if (ci)
            ZK_LAUNCH(ctx, k_colsum_rows<4>, R, 256, 0, M, N, rows, E2, partials, slots);
        else
            ZK_LAUNCH(ctx, k_colsum_rows<2>, R, 256, 0, M, N, rows, E2, partials, slots);
        ZK_LAUNCH(ctx, k_colsum_rows_finish, grid_for(ctx, N * cols, 256, 4), 256, 0, (const uint32_t*)partials, N, rows,
                  cols, R, slots, out);
        return;
    }
    // 128-thread CTAs, up to 7 resident per SM (70 registers): size the work to about one wave
    const uint64_t outputs = N * cols, slots = (uint64_t)ctx->num_sms * 7 * 128;
    uint32_t S = 1;
    while ((uint64_t)S * 2 * outputs <= slots && rows / (S * 2) >= 32 && rows % (S * 2) == 0) S *= 2;
    uint32_t* partials = S > 1 ? s.alloc<uint32_t>(outputs * S * 10) : nullptr;
    const uint64_t items = outputs * S;
    const uint64_t blocks = (items + 127) / 128;
    const unsigned int grid = (unsigned int)(blocks < (uint64_t)ctx->num_sms * 7 ? blocks : (uint64_t)ctx->num_sms * 7);
    ZK_LAUNCH(ctx, k_colsum_i32<LoadPlain>, grid, 128, 0, LoadPlain{M}, N, rows, cols, E2, out, S, partials);
    if (S > 1) ZK_LAUNCH(ctx, k_colsum_finish, grid_for(ctx, outputs, 256, 4), 256, 0, (const uint32_t*)partials, N, cols, S, out);
}

}  // namespace zk
