// restrict_tc.cu — the row dots of the matmul restriction (row a3) as an int8 GEMM on the
// 5th-generation tensor cores:   out[r] = sum_c M[r][c] E2[c]   for an int32 matrix M (rows x cols, row
// major) and Fr weights E2 (the eq table of u3 scaled by R, "double Montgomery", as k_rowdot_i32).
//
// With v = M[r][c] = b0 + 2^8 b1 + 2^16 b2 + 2^24 s3 (b_l unsigned bytes, s3 the signed top byte) and E2[c] =
// sum_q 2^{8q} e_q(c) (32 unsigned bytes), the integer X_r = sum_c v E2 = sum_{s < 35} 2^{8s} D_r[s] with
//     D_r[s] = sum_c ( sum_{l <= 2} b_l(r, c) e_{s-l}(c) + s3(r, c) e_{s-3}(c) ).
// The A operand is the raw bytes of M's rows (K index 4c + l: exactly the row-major memory), two MMAs per
// K step of 8 columns: A as u8 against B1[(c, l)][s] = [l <= 2] e_{s-l}(c), and A as s8 against
// B2[(c, l)][s] = [l = 3] e_{s-3}(c) (the lower bytes meet zero rows of B2, so their sign reading is moot).
// M = 128 rows per tile, N = 48 (35 shifts), K = 32 bytes; s32 accumulators in TMEM (|D| < 2^28 for
// cols <= 2^12).  The epilogue composes X_r + 2^31 S (S = sum_c E2[c], making the integer non-negative,
// as the CUDA-core kernel's u = v + 2^31 does), Montgomery-reduces and subtracts 2^31.
// CTA roles: warps 0-7 load each stage of RT_KS K steps (A: 128 rows x 32 B per K step with cp.async into the
// K-major core-matrix layout; B: the K steps' two 48 x 32-byte tiles of precomputed images) into a ring of
// stages; warp 8 issues the MMAs; warps 9-12 drain a double-buffered accumulator (warp w reads TMEM lanes
// 32 (w mod 4) ..).  Measured: ~2.2 TB/s from HBM with the tensor pipe 4.5% busy — the cp.async loads are
// latency-bound: every stage reads a 128 B (RT_KS = 4) piece of 4 KB-strided rows; 3 stages of 8 K steps
// (256 B of every row per stage) cut the window's row dots 0.74 -> 0.67 ms (serial kernel tables).  A TMA
// (128-byte swizzle) producer is the next step (a first attempt stalled when a CTA owned several tiles).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>

#include "tables.cuh"
#include "tc.cuh"

namespace zk {

constexpr int RT_STAGES = 3;
constexpr int RT_KS = 8;                  // K steps (of 8 columns, 32 bytes) per pipeline stage: 256 B of every row
constexpr int RT_ABYTES = 128 * 32;       // one K step of A
constexpr int RT_BBYTES = 48 * 32;        // one K step of one B part
constexpr uint32_t RT_IDESC_U = (2u << 4) | ((48u >> 3) << 17) | ((128u >> 4) << 24);   // s32 += u8 x u8
constexpr uint32_t RT_IDESC_S = RT_IDESC_U | (1u << 7);                                  // s32 += s8 x u8
constexpr int RT_THREADS = 13 * 32;

struct __align__(1024) RtSmem {
    uint8_t A[RT_STAGES][RT_KS][RT_ABYTES];
    uint8_t B[RT_STAGES][RT_KS][2][RT_BBYTES];
    uint64_t full[RT_STAGES], empty[RT_STAGES], accfull[2], accempty[2];
    uint32_t tmem;
};

// byte offset of (row, byte k) in a K-major, no-swizzle tile of 8-row x 16-byte core matrices
// (LBO = 128 B between the two 16-byte K chunks, SBO = 256 B between 8-row groups; see bdesc)
__device__ __forceinline__ uint32_t rt_off(uint32_t row, uint32_t kb) {
    return (row >> 3) * 256 + (kb >> 4) * 128 + (row & 7) * 16 + (kb & 15);
}

// B images for every K step: Bimg[ks][part][rt_off(n, kb)], part 0 = the u8 tile, 1 = the s8 tile
__global__ void k_rt_bimg(const fr_t* E2, uint32_t cols, uint8_t* Bimg) {
    const uint64_t total = (uint64_t)(cols / 8) * 2 * 48 * 32;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total; g += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t kb = g % 32, n = (g / 32) % 48, part = (g / (32 * 48)) % 2;
        const uint64_t ks = g / (32 * 48 * 2);
        const uint32_t c = (uint32_t)(ks * 8 + kb / 4), l = kb % 4;
        int q = (int)n - (int)l;
        uint8_t v = 0;
        if (q >= 0 && q < 32 && (part ? l == 3 : l <= 2)) {
            const uint32_t limb = __ldg(&E2[c].v[q >> 2]);
            v = (uint8_t)(limb >> (8 * (q & 3)));
        }
        Bimg[(ks * 2 + part) * RT_BBYTES + rt_off(n, kb)] = v;
    }
}

// bias = 2^31 * S, S = sum_c E2[c] as an integer (< 2^268 for cols <= 2^12), as 10 little-endian limbs;
// one block of 1024 threads (word sums by warp shuffles, then across warps)
__global__ void __launch_bounds__(1024) k_rt_bias(const fr_t* E2, uint32_t cols, uint32_t* bias) {
    __shared__ uint64_t part[32][8];
    uint64_t a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint32_t c = threadIdx.x; c < cols; c += blockDim.x) {
        const fr_t e = fr_load(&E2[c]);
#pragma unroll
        for (int i = 0; i < 8; i++) a[i] += e.v[i];   // word sums < 2^44
    }
#pragma unroll
    for (int i = 0; i < 8; i++)
        for (int off = 16; off > 0; off >>= 1) a[i] += __shfl_down_sync(0xffffffffu, a[i], off);
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int i = 0; i < 8; i++) part[threadIdx.x >> 5][i] = a[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t sw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int t = 0; t < (int)(blockDim.x >> 5); t++)
            for (int i = 0; i < 8; i++) sw[i] += part[t][i];
        uint32_t w[10];
        uint64_t carry = 0;
        for (int i = 0; i < 10; i++) {   // normalise to 32-bit limbs
            const uint64_t v = (i < 8 ? sw[i] : 0ull) + carry;
            w[i] = (uint32_t)v;
            carry = v >> 32;
        }
        for (int i = 0; i < 10; i++) bias[i] = (w[i] << 31) | (i ? (w[i - 1] >> 1) : 0u);   // S << 31
    }
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(dst)), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void mma_i8_ss(uint32_t d, uint64_t adesc, uint64_t bdesc_, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(adesc), "l"(bdesc_), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// mbarrier wait with a watchdog (diagnostics: a lost arrival traps with the barrier's name instead of hanging)
__device__ __forceinline__ void rt_wait(uint64_t* b, uint32_t parity, int id) {
    uint32_t done = 0;
    uint64_t n = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(su32(b)), "r"(parity)
            : "memory");
        if (++n == (1ull << 26)) {
            printf("k_rowdot_tc: stuck on barrier %d parity %u (block %d thread %d)\n", id, parity, blockIdx.x, threadIdx.x);
            __trap();
        }
    }
}

struct RtArgs {
    const int32_t* M;
    uint64_t nrows;
    uint32_t cols;
    const uint8_t* Bimg;
    const uint32_t* bias;
    fr_t* out;
    uint64_t inner, outer;
    uint32_t log_inner;
};

__global__ void __launch_bounds__(RT_THREADS, 1) k_rowdot_tc(RtArgs a) {
    extern __shared__ __align__(1024) uint8_t rt_raw[];
    RtSmem& S = *reinterpret_cast<RtSmem*>(rt_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t KS = a.cols / 8;
    const uint64_t ntiles = (a.nrows + 127) / 128;
    if (warp == 8) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&S.tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        if (lane == 0) {
            for (int i = 0; i < RT_STAGES; i++) {
                mbar_init(&S.full[i], 256);
                mbar_init(&S.empty[i], 1);
            }
            for (int i = 0; i < 2; i++) {
                mbar_init(&S.accfull[i], 1);
                mbar_init(&S.accempty[i], 4);
            }
            asm volatile("fence.mbarrier_init.release.cluster;");
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem;
    if (warp < 8) {
        // ---------------- producers: per stage RT_KS K steps; thread t loads A chunks (row t / 2, 16-byte
        // half t % 2) of every K step and B chunks t, t + 256, ... of the stage's RT_KS x 3 KB image
        const uint32_t t = threadIdx.x;
        const uint32_t arow = t >> 1, akc = t & 1;
        const uint32_t KSS = (KS + RT_KS - 1) / RT_KS;   // stages per tile
        uint64_t it = 0;
        for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const uint64_t row = tile * 128 + arow;
            const bool in = row < a.nrows;
            const uint8_t* srow = reinterpret_cast<const uint8_t*>(a.M + (in ? row : 0) * (uint64_t)a.cols);
            for (uint32_t sg = 0; sg < KSS; sg++, it++) {
                const uint32_t st = it % RT_STAGES;
                if (it >= RT_STAGES) rt_wait(&S.empty[st], ((it / RT_STAGES) - 1) & 1, 1);
                const uint32_t k0 = sg * RT_KS, nk = KS - k0 < (uint32_t)RT_KS ? KS - k0 : (uint32_t)RT_KS;
#pragma unroll
                for (int kk = 0; kk < RT_KS; kk++)
                    if ((uint32_t)kk < nk)
                        cp_async16(&S.A[st][kk][rt_off(arow, akc * 16)], srow + (k0 + kk) * 32 + akc * 16, in ? 16u : 0u);
                const uint8_t* bsrc = a.Bimg + (uint64_t)k0 * 2 * RT_BBYTES;
                for (uint32_t c16 = t; c16 < nk * 2 * RT_BBYTES / 16; c16 += 256)
                    cp_async16(&S.B[st][0][0][c16 * 16], bsrc + c16 * 16, 16u);
                asm volatile("cp.async.commit_group;" ::: "memory");
                if (it >= RT_STAGES - 1) {   // the stage issued RT_STAGES - 1 stages ago has landed: publish it
                    asm volatile("cp.async.wait_group %0;" ::"n"(RT_STAGES - 1) : "memory");
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_arrive(&S.full[(it - (RT_STAGES - 1)) % RT_STAGES]);
                }
            }
        }
        // drain: publish the last RT_STAGES - 1 stages
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint64_t first = it >= (uint64_t)(RT_STAGES - 1) ? it - (RT_STAGES - 1) : 0;
        for (uint64_t j = first; j < it; j++) mbar_arrive(&S.full[j % RT_STAGES]);
    } else if (warp == 8) {
        // ---------------- MMA issuer
        const uint32_t KSS = (KS + RT_KS - 1) / RT_KS;
        uint64_t it = 0, ti = 0;
        for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ti++) {
            const uint32_t buf = ti & 1;
            if (ti >= 2) rt_wait(&S.accempty[buf], ((ti / 2) - 1) & 1, 2);
            tc_fence_after();
            for (uint32_t sg = 0; sg < KSS; sg++, it++) {
                const uint32_t st = it % RT_STAGES;
                rt_wait(&S.full[st], (it / RT_STAGES) & 1, 3);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t k0 = sg * RT_KS, nk = KS - k0 < (uint32_t)RT_KS ? KS - k0 : (uint32_t)RT_KS;
                    for (uint32_t kk = 0; kk < nk; kk++) {
                        const uint64_t ad = bdesc(S.A[st][kk]);
                        mma_i8_ss(tmem + 64 * buf, ad, bdesc(S.B[st][kk][0]), RT_IDESC_U, (k0 + kk) > 0);
                        mma_i8_ss(tmem + 64 * buf, ad, bdesc(S.B[st][kk][1]), RT_IDESC_S, 1u);
                    }
                    mma_commit(&S.empty[st]);
                    if (sg + 1 == KSS) mma_commit(&S.accfull[buf]);
                }
                __syncwarp();
            }
        }
    } else {
        // ---------------- epilogue: warp w drains TMEM lanes 32 (w mod 4) .. + 31
        const uint32_t q = warp & 3;
        uint32_t bias[10];
#pragma unroll
        for (int i = 0; i < 10; i++) bias[i] = __ldg(&a.bias[i]);
        uint64_t ti = 0;
        for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ti++) {
            const uint32_t buf = ti & 1;
            rt_wait(&S.accfull[buf], (ti / 2) & 1, 4);
            tc_fence_after();
            uint32_t d[40];
            const uint32_t taddr = tmem + ((32 * q) << 16) + 64 * buf;
            {
                uint32_t v32[32];
                tmem_ld32(taddr, v32);
#pragma unroll
                for (int i = 0; i < 32; i++) d[i] = v32[i];
                uint32_t v8[8];
                tmem_ld8(taddr + 32, v8);
#pragma unroll
                for (int i = 0; i < 8; i++) d[32 + i] = v8[i];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.accempty[buf]);
            const uint64_t row = tile * 128 + 32 * q + lane;
            if (row < a.nrows) {
                int64_t acc[10];
#pragma unroll
                for (int i = 0; i < 10; i++) acc[i] = (int64_t)bias[i];
#pragma unroll
                for (int s = 0; s < 35; s++) acc[s >> 2] += (int64_t)(int32_t)d[s] << (8 * (s & 3));
                uint32_t w[10];
                int64_t carry = 0;
#pragma unroll
                for (int i = 0; i < 10; i++) {
                    const int64_t v = acc[i] + carry;
                    w[i] = (uint32_t)v;
                    carry = v >> 32;   // arithmetic: partial sums may be negative before the bias settles
                }
                const uint64_t o = (row & (a.inner - 1)) * a.outer + (row >> a.log_inner);
                fr_store(&a.out[o], wide_finish(w));
            }
        }
    }
    __syncthreads();
    if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

// ---------------------------------------------------------------- the TMA producer (round 2)
// The same GEMM with the A operand moved by the tensor-memory accelerator: a 2D tensor map over M's bytes
// (rows x 4 cols), boxes of 128 rows x 128 bytes (4 K steps) in the 128-byte-swizzled K-major layout the
// MMA reads directly (SW128 descriptor, SBO = 1024 B; the K step within a box advances the start address by
// 32 B); rows past the end and bytes past a row are zero-filled by the TMA unit.  One thread issues a
// stage (two boxes + one bulk copy of the B images) against one transaction-counted barrier, so the
// producer costs no issue slots; the MMA and epilogue warps are the kernel above.
constexpr int RM_STAGES = 3;
struct __align__(1024) RmSmem {
    uint8_t A[RM_STAGES][RT_KS / 4][128 * 128];
    uint8_t B[RM_STAGES][RT_KS][2][RT_BBYTES];
    uint64_t full[RM_STAGES], empty[RM_STAGES], accfull[2], accempty[2];
    uint32_t tmem;
};

__device__ __forceinline__ uint64_t adesc_sw128(const void* p) {
    return (uint64_t)((su32(p) >> 4) & 0x3fff) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t x, int32_t y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(bar))
        : "memory");
}

__global__ void __launch_bounds__(RT_THREADS, 1) k_rowdot_tma(RtArgs a, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(1024) uint8_t rm_raw[];
    RmSmem& S = *reinterpret_cast<RmSmem*>(rm_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t KS = a.cols / 8;
    const uint32_t KSS = (KS + RT_KS - 1) / RT_KS;
    const uint64_t ntiles = (a.nrows + 127) / 128;
    if (warp == 8) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&S.tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        if (lane == 0) {
            for (int i = 0; i < RM_STAGES; i++) {
                mbar_init(&S.full[i], 1);
                mbar_init(&S.empty[i], 1);
            }
            for (int i = 0; i < 2; i++) {
                mbar_init(&S.accfull[i], 1);
                mbar_init(&S.accempty[i], 4);
            }
            asm volatile("fence.mbarrier_init.release.cluster;");
        }
    }
    if (warp == 0 && lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem;
    if (warp == 0) {
        // ---------------- producer: one thread, one barrier transaction per stage
        if (lane == 0) {
            uint64_t it = 0;
            for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (uint32_t sg = 0; sg < KSS; sg++, it++) {
                    const uint32_t st = it % RM_STAGES;
                    if (it >= RM_STAGES) rt_wait(&S.empty[st], ((it / RM_STAGES) - 1) & 1, 11);
                    const uint32_t k0 = sg * RT_KS, nk = KS - k0 < (uint32_t)RT_KS ? KS - k0 : (uint32_t)RT_KS;
                    const uint32_t nbox = (nk + 3) / 4;
                    mbar_expect_tx(&S.full[st], nbox * 128 * 128 + nk * 2 * RT_BBYTES);
                    for (uint32_t b = 0; b < nbox; b++)
                        tma_load_2d(S.A[st][b], &tmap, (int32_t)((k0 + 4 * b) * 32), (int32_t)(tile * 128), &S.full[st]);
                    bulk_g2s(S.B[st][0][0], a.Bimg + (uint64_t)k0 * 2 * RT_BBYTES, nk * 2 * RT_BBYTES, &S.full[st]);
                }
            }
        }
    } else if (warp == 8) {
        // ---------------- MMA issuer
        uint64_t it = 0, ti = 0;
        for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ti++) {
            const uint32_t buf = ti & 1;
            if (ti >= 2) rt_wait(&S.accempty[buf], ((ti / 2) - 1) & 1, 12);
            tc_fence_after();
            for (uint32_t sg = 0; sg < KSS; sg++, it++) {
                const uint32_t st = it % RM_STAGES;
                rt_wait(&S.full[st], (it / RM_STAGES) & 1, 13);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t k0 = sg * RT_KS, nk = KS - k0 < (uint32_t)RT_KS ? KS - k0 : (uint32_t)RT_KS;
                    for (uint32_t kk = 0; kk < nk; kk++) {
                        const uint64_t ad = adesc_sw128(S.A[st][kk >> 2] + 32 * (kk & 3));
                        mma_i8_ss(tmem + 64 * buf, ad, bdesc(S.B[st][kk][0]), RT_IDESC_U, (k0 + kk) > 0);
                        mma_i8_ss(tmem + 64 * buf, ad, bdesc(S.B[st][kk][1]), RT_IDESC_S, 1u);
                    }
                    mma_commit(&S.empty[st]);
                    if (sg + 1 == KSS) mma_commit(&S.accfull[buf]);
                }
                __syncwarp();
            }
        }
    } else if (warp >= 9) {
        // ---------------- epilogue: warp w drains TMEM lanes 32 (w mod 4) .. + 31
        const uint32_t q = warp & 3;
        uint32_t bias[10];
#pragma unroll
        for (int i = 0; i < 10; i++) bias[i] = __ldg(&a.bias[i]);
        uint64_t ti = 0;
        for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ti++) {
            const uint32_t buf = ti & 1;
            rt_wait(&S.accfull[buf], (ti / 2) & 1, 14);
            tc_fence_after();
            uint32_t d[40];
            const uint32_t taddr = tmem + ((32 * q) << 16) + 64 * buf;
            {
                uint32_t v32[32];
                tmem_ld32(taddr, v32);
#pragma unroll
                for (int i = 0; i < 32; i++) d[i] = v32[i];
                uint32_t v8[8];
                tmem_ld8(taddr + 32, v8);
#pragma unroll
                for (int i = 0; i < 8; i++) d[32 + i] = v8[i];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.accempty[buf]);
            const uint64_t row = tile * 128 + 32 * q + lane;
            if (row < a.nrows) {
                int64_t acc[10];
#pragma unroll
                for (int i = 0; i < 10; i++) acc[i] = (int64_t)bias[i];
#pragma unroll
                for (int s = 0; s < 35; s++) acc[s >> 2] += (int64_t)(int32_t)d[s] << (8 * (s & 3));
                uint32_t w[10];
                int64_t carry = 0;
#pragma unroll
                for (int i = 0; i < 10; i++) {
                    const int64_t v = acc[i] + carry;
                    w[i] = (uint32_t)v;
                    carry = v >> 32;
                }
                const uint64_t o = (row & (a.inner - 1)) * a.outer + (row >> a.log_inner);
                fr_store(&a.out[o], wide_finish(w));
            }
        }
    }
    __syncthreads();
    if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 1: the TMA producer (default), 0: the cp.async producer (ZKDL_ROWDOT_TMA=0)
static bool rowdot_tma_on() {
    static const bool off = getenv("ZKDL_ROWDOT_TMA") && atoi(getenv("ZKDL_ROWDOT_TMA")) == 0;
    return !off;
}

static void rowdot_tma_launch(zk_ctx* ctx, const RtArgs& a) {
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    ZK_REQUIRE(enc != nullptr, ZK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)a.cols * 4, (cuuint64_t)a.nrows};
    const cuuint64_t strides[1] = {(cuuint64_t)a.cols * 4};
    const cuuint32_t box[2] = {128, 128};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int32_t*>(a.M), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    ZK_REQUIRE(r == CUDA_SUCCESS, ZK_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    const size_t smem = sizeof(RmSmem) + 1024;
    static bool attr = false;
    if (!attr) {
        ZK_CUDA(cudaFuncSetAttribute(k_rowdot_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    const uint64_t ntiles = (a.nrows + 127) / 128;
    const unsigned int grid = (unsigned int)(ntiles < (uint64_t)ctx->num_sms ? ntiles : (uint64_t)ctx->num_sms);
    ZK_LAUNCH(ctx, k_rowdot_tma, grid, RT_THREADS, smem, a, map);
}

// ---------------------------------------------------------------- column sums on the tensor cores (round 2)
// out[c * N + n] = sum_r E2[r] M[n][r][c] (colsum_i32) for an int32 stack M[N][rows][cols]: the contraction
// index r is the row index of the stored matrix, so the A operand is MN-major — M = 128 byte columns
// (32 int32 columns x 4 byte positions, contiguous in memory), K = 32 matrix rows — and the TMA unit moves
// it untransformed: a box of 32 rows x 128 bytes with 128-byte swizzle is exactly the MN-major SW128 layout
// (instruction descriptor bit 15; validated by scripts/tc_mn_probe.cu for u8 and s8).  B = the 32 limb bytes
// of E2 for those 32 rows (K-major, one 1 KB image per K step), N = 32:
//     D[4 c + l][q] = sum_r byte_l(M[n][r][c]) e_q(r),   X_c = sum_{l, q} 2^{8 (l + q)} D[4 c + l][q]
// with the top byte signed (a second MMA reads A as s8; lane 4c+3 takes that result).  |D| < rows 2^16, so
// rows <= 4096.  The epilogue forms each lane's 320-bit two's-complement partial, shifts it by 8 l, adds the
// four byte lanes of a column by shuffles, adds the bias 2^31 S (S = sum_r E2[r]) and reduces (wide_finish),
// as k_colsum_i32 does with u = v + 2^31.  Roles: warp 0 the TMA producer, warp 1 the MMA issuer, warps 2-5
// the epilogue over a double-buffered accumulator (64 TMEM columns each: u8 result, s8 result).
constexpr int CT_SKS = 8;                  // K steps (32 rows each) per stage
constexpr int CT_STAGES = 4;
constexpr uint32_t CT_IDESC_U = (2u << 4) | (1u << 15) | ((32u >> 3) << 17) | ((128u >> 4) << 24);   // A MN-major
constexpr uint32_t CT_IDESC_S = CT_IDESC_U | (1u << 7);
constexpr int CT_THREADS = 6 * 32;

struct __align__(1024) CtSmem {
    uint8_t A[CT_STAGES][CT_SKS][32 * 128];
    uint8_t B[CT_STAGES][CT_SKS][1024];
    uint64_t full[CT_STAGES], empty[CT_STAGES], accfull[2], accempty[2];
    uint32_t tmem;
};

struct CtArgs {
    uint64_t N;
    uint32_t rows, cols;
    const uint8_t* Bimg;     // [rows / 32][1024]: limb q of E2[32 ks + kb] at rt_off(q, kb)
    const uint32_t* bias;
    fr_t* out;
};

// B images of the column sums: K step ks holds E2[32 ks .. 32 ks + 31] as 32 limb rows (K-major, no swizzle)
__global__ void k_ct_bimg(const fr_t* E2, uint32_t rows, uint8_t* Bimg) {
    const uint64_t total = (uint64_t)rows * 32;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total; g += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = (uint32_t)(g % 32), r = (uint32_t)(g / 32);
        const uint32_t limb = __ldg(&E2[r].v[q >> 2]);
        Bimg[(uint64_t)(r / 32) * 1024 + rt_off(q, r % 32)] = (uint8_t)(limb >> (8 * (q & 3)));
    }
}

__global__ void __launch_bounds__(CT_THREADS, 1) k_colsum_tma(CtArgs a, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(1024) uint8_t ct_raw[];
    CtSmem& S = *reinterpret_cast<CtSmem*>(ct_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t KS = a.rows / 32, KSS = (KS + CT_SKS - 1) / CT_SKS, CB = a.cols / 32;
    const uint64_t ntiles = a.N * CB;
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&S.tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        if (lane == 0) {
            for (int i = 0; i < CT_STAGES; i++) {
                mbar_init(&S.full[i], 1);
                mbar_init(&S.empty[i], 1);
            }
            for (int i = 0; i < 2; i++) {
                mbar_init(&S.accfull[i], 1);
                mbar_init(&S.accempty[i], 4);
            }
            asm volatile("fence.mbarrier_init.release.cluster;");
        }
    }
    if (warp == 0 && lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem;
    if (warp == 0) {
        // ---------------- producer: one thread, one transaction-counted barrier per stage
        if (lane == 0) {
            uint64_t it = 0;
            for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const uint64_t n = tile / CB, cb = tile % CB;
                for (uint32_t sg = 0; sg < KSS; sg++, it++) {
                    const uint32_t st = it % CT_STAGES;
                    if (it >= CT_STAGES) rt_wait(&S.empty[st], ((it / CT_STAGES) - 1) & 1, 21);
                    const uint32_t k0 = sg * CT_SKS, nk = KS - k0 < (uint32_t)CT_SKS ? KS - k0 : (uint32_t)CT_SKS;
                    mbar_expect_tx(&S.full[st], nk * (32 * 128 + 1024));
                    for (uint32_t kk = 0; kk < nk; kk++)
                        tma_load_2d(S.A[st][kk], &tmap, (int32_t)(cb * 128), (int32_t)(n * a.rows + 32 * (k0 + kk)), &S.full[st]);
                    bulk_g2s(S.B[st][0], a.Bimg + (uint64_t)k0 * 1024, nk * 1024, &S.full[st]);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        uint64_t it = 0, ti = 0;
        for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ti++) {
            const uint32_t buf = ti & 1;
            if (ti >= 2) rt_wait(&S.accempty[buf], ((ti / 2) - 1) & 1, 22);
            tc_fence_after();
            for (uint32_t sg = 0; sg < KSS; sg++, it++) {
                const uint32_t st = it % CT_STAGES;
                rt_wait(&S.full[st], (it / CT_STAGES) & 1, 23);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t k0 = sg * CT_SKS, nk = KS - k0 < (uint32_t)CT_SKS ? KS - k0 : (uint32_t)CT_SKS;
                    for (uint32_t kk = 0; kk < nk; kk++) {
                        const uint64_t ad = adesc_sw128(S.A[st][kk]), bd = bdesc(S.B[st][kk]);
                        mma_i8_ss(tmem + 64 * buf, ad, bd, CT_IDESC_U, (k0 + kk) > 0);
                        mma_i8_ss(tmem + 64 * buf + 32, ad, bd, CT_IDESC_S, (k0 + kk) > 0);
                    }
                    mma_commit(&S.empty[st]);
                    if (sg + 1 == KSS) mma_commit(&S.accfull[buf]);
                }
                __syncwarp();
            }
        }
    } else {
        // ---------------- epilogue: warp w drains TMEM lanes 32 (w mod 4) .. + 31 (lane = byte column 4 c + l)
        const uint32_t q = warp & 3, l = lane & 3;
        uint32_t bias[10];
#pragma unroll
        for (int i = 0; i < 10; i++) bias[i] = l == 0 ? __ldg(&a.bias[i]) : 0u;
        uint64_t ti = 0;
        for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ti++) {
            const uint32_t buf = ti & 1;
            rt_wait(&S.accfull[buf], (ti / 2) & 1, 24);
            tc_fence_after();
            uint32_t d[32];
            {
                const uint32_t taddr = tmem + ((32 * q) << 16) + 64 * buf;
                uint32_t du[32], ds[32];
                tmem_ld32(taddr, du);
                tmem_ld32(taddr + 32, ds);
#pragma unroll
                for (int i = 0; i < 32; i++) d[i] = l == 3 ? ds[i] : du[i];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.accempty[buf]);
            // this lane's partial sum_q 2^{8 q} D[q] as 320-bit two's complement
            int64_t acc[10];
#pragma unroll
            for (int i = 0; i < 10; i++) acc[i] = 0;
#pragma unroll
            for (int s = 0; s < 32; s++) acc[s >> 2] += (int64_t)(int32_t)d[s] << (8 * (s & 3));
            uint32_t w[10];
            int64_t carry = 0;
#pragma unroll
            for (int i = 0; i < 10; i++) {
                const int64_t v = acc[i] + carry;
                w[i] = (uint32_t)v;
                carry = v >> 32;
            }
            // times 2^{8 l}, then the four byte lanes of the column added by shuffles (mod 2^320), + bias
            if (l) {
                const uint32_t sh = 8 * l;
#pragma unroll
                for (int i = 9; i > 0; i--) w[i] = (w[i] << sh) | (w[i - 1] >> (32 - sh));
                w[0] <<= sh;
            }
            uint32_t c0 = 0;
#pragma unroll
            for (int i = 0; i < 10; i++) {   // + bias (lane l = 0 only; the others add zero)
                const uint64_t v = (uint64_t)w[i] + bias[i] + c0;
                w[i] = (uint32_t)v;
                c0 = (uint32_t)(v >> 32);
            }
#pragma unroll
            for (int off = 1; off <= 2; off <<= 1) {
                uint32_t o[10];
#pragma unroll
                for (int i = 0; i < 10; i++) o[i] = __shfl_xor_sync(0xffffffffu, w[i], off);
                uint32_t cc = 0;
#pragma unroll
                for (int i = 0; i < 10; i++) {
                    const uint64_t v = (uint64_t)w[i] + o[i] + cc;
                    w[i] = (uint32_t)v;
                    cc = (uint32_t)(v >> 32);
                }
            }
            if (l == 0) {
                const uint64_t n = tile / CB, c = (tile % CB) * 32 + 8 * q + (lane >> 2);
                fr_store(&a.out[c * a.N + n], wide_finish(w));
            }
        }
    }
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

bool colsum_tc_ok(uint64_t N, uint32_t rows, uint32_t cols) {
    static const bool off = getenv("ZKDL_COLSUM_TC") && atoi(getenv("ZKDL_COLSUM_TC")) == 0;
    return !off && cols % 32 == 0 && rows % 32 == 0 && rows >= 32 && rows <= 4096 && N * (cols / 32) >= 148 &&
           N * rows * 4ull * cols >= (8ull << 20);
}

void colsum_tc(zk_ctx* ctx, const int32_t* M, uint64_t N, uint32_t rows, uint32_t cols, const fr_t* E2, fr_t* out,
               Scratch& s) {
    uint8_t* Bimg = s.alloc<uint8_t>((size_t)rows * 32);
    ZK_LAUNCH(ctx, k_ct_bimg, grid_for(ctx, (uint64_t)rows * 32, 256, 4), 256, 0, E2, rows, Bimg);
    uint32_t* bias = s.alloc<uint32_t>(10);
    ZK_LAUNCH(ctx, k_rt_bias, 1, 1024, 0, E2, rows, bias);
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    ZK_REQUIRE(enc != nullptr, ZK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)cols * 4, (cuuint64_t)N * rows};
    const cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    const cuuint32_t box[2] = {128, 32};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int32_t*>(M), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    ZK_REQUIRE(r == CUDA_SUCCESS, ZK_ERR_CUDA, "cuTensorMapEncodeTiled failed (column sums)");
    CtArgs a;
    a.N = N;
    a.rows = rows;
    a.cols = cols;
    a.Bimg = Bimg;
    a.bias = bias;
    a.out = out;
    const size_t smem = sizeof(CtSmem) + 1024;
    static bool attr = false;
    if (!attr) {
        ZK_CUDA(cudaFuncSetAttribute(k_colsum_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    const uint64_t ntiles = N * (cols / 32);
    const unsigned int grid = (unsigned int)(ntiles < (uint64_t)ctx->num_sms ? ntiles : (uint64_t)ctx->num_sms);
    ZK_LAUNCH(ctx, k_colsum_tma, grid, CT_THREADS, smem, a, map);
}

bool rowdot_tc_ok(uint64_t nrows, uint32_t cols) {
    static const bool off = getenv("ZKDL_ROWDOT_TC") && atoi(getenv("ZKDL_ROWDOT_TC")) == 0;
    return !off && cols % 8 == 0 && cols >= 8 && cols <= 4096 && nrows >= 1024;
}

void rowdot_tc(zk_ctx* ctx, const int32_t* M, uint64_t nrows, uint32_t cols, const fr_t* E2, fr_t* out, uint64_t inner,
               uint32_t log_inner, uint64_t outer, Scratch& s, int use_tma) {
    const uint32_t KS = cols / 8;
    uint8_t* Bimg = s.alloc<uint8_t>((size_t)KS * 2 * RT_BBYTES);
    ZK_LAUNCH(ctx, k_rt_bimg, grid_for(ctx, (uint64_t)KS * 2 * RT_BBYTES, 256, 4), 256, 0, E2, cols, Bimg);
    uint32_t* bias = s.alloc<uint32_t>(10);
    ZK_LAUNCH(ctx, k_rt_bias, 1, 1024, 0, E2, cols, bias);
    RtArgs a;
    a.M = M;
    a.nrows = nrows;
    a.cols = cols;
    a.Bimg = Bimg;
    a.bias = bias;
    a.out = out;
    a.inner = inner;
    a.outer = outer;
    a.log_inner = log_inner;
    if (use_tma < 0 ? rowdot_tma_on() : use_tma != 0) {
        rowdot_tma_launch(ctx, a);
        return;
    }
    const size_t smem = sizeof(RtSmem) + 1024;
    static bool attr = false;
    if (!attr) {
        ZK_CUDA(cudaFuncSetAttribute(k_rowdot_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    const uint64_t ntiles = (nrows + 127) / 128;
    const unsigned int grid = (unsigned int)(ntiles < (uint64_t)ctx->num_sms ? ntiles : (uint64_t)ctx->num_sms);
    ZK_LAUNCH(ctx, k_rowdot_tc, grid, RT_THREADS, smem, a);
}

}  // namespace zk
