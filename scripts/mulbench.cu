// Standalone Fr-multiplication microbenchmark (variants of the Montgomery product on sm_100a).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mulbench scripts/mulbench.cu && ./mulbench
// Prints G Fr-mul/s per variant and checks every variant against the production fr_mul.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../paper_2307_16273_b200/csrc/fr.cuh"

using namespace zk;

__device__ __constant__ uint32_t PC[8] = {ZK_P0, ZK_P1, ZK_P2, ZK_P3, ZK_P4, ZK_P5, ZK_P6, ZK_P7};

// Variant B: CIOS with 64-bit C intermediates (compiler-managed carries, no inline PTX).
__device__ __forceinline__ fr_t mul_u64(const fr_t& a, const fr_t& b) {
    const uint32_t p[8] = {ZK_P0, ZK_P1, ZK_P2, ZK_P3, ZK_P4, ZK_P5, ZK_P6, ZK_P7};
    uint32_t t[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint64_t C = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            uint64_t uv = (uint64_t)a.v[j] * b.v[i] + t[j] + C;
            t[j] = (uint32_t)uv;
            C = uv >> 32;
        }
        t[8] += (uint32_t)C;
        const uint32_t m = t[0] * 0xffffffffu;
        C = ((uint64_t)m * p[0] + t[0]) >> 32;
#pragma unroll
        for (int j = 1; j < 8; j++) {
            uint64_t uv = (uint64_t)m * p[j] + t[j] + C;
            t[j - 1] = (uint32_t)uv;
            C = uv >> 32;
        }
        uint64_t uv = (uint64_t)t[8] + C;
        t[7] = (uint32_t)uv;
        t[8] = (uint32_t)(uv >> 32);
    }
    fr_t r;
#pragma unroll
    for (int i = 0; i < 8; i++) r.v[i] = t[i];
    return fr_reduce_once(r);
}

// Variant C: separated operand scanning — full 512-bit product with 64-bit column accumulators of
// 32-bit half-products (no carry chains: sums of <= 16 terms < 2^36), then Montgomery reduction.
__device__ __forceinline__ fr_t mul_sos(const fr_t& a, const fr_t& b) {
    const uint32_t p[8] = {ZK_P0, ZK_P1, ZK_P2, ZK_P3, ZK_P4, ZK_P5, ZK_P6, ZK_P7};
    uint64_t col[17];
#pragma unroll
    for (int k = 0; k < 17; k++) col[k] = 0;
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) {
            uint64_t pr = (uint64_t)a.v[i] * b.v[j];
            col[i + j] += (uint32_t)pr;
            col[i + j + 1] += pr >> 32;
        }
    // montgomery: for i < 8: normalise column i, m = col_i * n0, add m*p
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const uint32_t ti = (uint32_t)col[i];
        col[i + 1] += col[i] >> 32;
        const uint32_t m = ti * 0xffffffffu;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            uint64_t pr = (uint64_t)m * p[j];
            col[i + j] += (uint32_t)pr;
            col[i + j + 1] += pr >> 32;
        }
        col[i + 1] += col[i] >> 32;   // col[i] low 32 bits are zero now
    }
    fr_t r;
    uint64_t c = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        uint64_t v = col[8 + k] + c;
        r.v[k] = (uint32_t)v;
        c = v >> 32;
    }
    return fr_reduce_once(r);
}

// Variant D: u64 CIOS using p0 = 1 and p1 = 2^32 - 1 in the reduction (m p1 = (m << 32) - m on the
// ALU pipe instead of an IMAD.WIDE on the FMA pipe).
__device__ __forceinline__ fr_t mul_u64p(const fr_t& a, const fr_t& b) {
    const uint32_t p[8] = {ZK_P0, ZK_P1, ZK_P2, ZK_P3, ZK_P4, ZK_P5, ZK_P6, ZK_P7};
    uint32_t t[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint64_t C = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            uint64_t uv = (uint64_t)a.v[j] * b.v[i] + t[j] + C;
            t[j] = (uint32_t)uv;
            C = uv >> 32;
        }
        t[8] += (uint32_t)C;
        const uint32_t m = t[0] * 0xffffffffu;   // = -t0
        // j = 0: t0 + m*1 = 0 mod 2^32 with carry (t0 != 0)
        C = (uint64_t)(t[0] != 0);
        // j = 1: m*(2^32-1) + t1 + C = (m << 32) + t1 + C - m
        {
            uint64_t uv = ((uint64_t)m << 32) + t[1] + C - m;
            t[0] = (uint32_t)uv;
            C = uv >> 32;
        }
#pragma unroll
        for (int j = 2; j < 8; j++) {
            uint64_t uv = (uint64_t)m * p[j] + t[j] + C;
            t[j - 1] = (uint32_t)uv;
            C = uv >> 32;
        }
        uint64_t uv = (uint64_t)t[8] + C;
        t[7] = (uint32_t)uv;
        t[8] = (uint32_t)(uv >> 32);
    }
    fr_t r;
#pragma unroll
    for (int i = 0; i < 8; i++) r.v[i] = t[i];
    return fr_reduce_once(r);
}

// Variant E: a*b_i rows with 64-bit compiler carries (FMA + ALU pipes), reduction rows as PTX madc
// chains (FMA pipe only) -- balances the two pipes.
__device__ __forceinline__ fr_t mul_mix(const fr_t& a, const fr_t& b) {
    uint32_t t[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint64_t C = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            uint64_t uv = (uint64_t)a.v[j] * b.v[i] + t[j] + C;
            t[j] = (uint32_t)uv;
            C = uv >> 32;
        }
        t[8] += (uint32_t)C;
        ZK_REDC_ROW(t);
    }
    fr_t r;
#pragma unroll
    for (int i = 0; i < 8; i++) r.v[i] = t[i];
    return fr_reduce_once(r);
}

// Variant F: production product without the final conditional subtraction (output < 2p; valid as an
// input to the next product because 4p < 2^256).
__device__ __forceinline__ fr_t mul_lazy(const fr_t& a, const fr_t& b) {
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
        const uint32_t m = t[0] * 0xffffffffu;
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
    return r;
}

// Variant 8: the production CIOS with every carry folded into the 64-bit addend of the product
// (x + C as a 33-bit value from PTX add.cc / addc, meant for the ALU pipe), so IMAD.WIDE.U32 carries no
// separate high-word carry add (the IMAD.X the compiler puts on the FMA pipe)
__device__ __forceinline__ uint64_t add33(uint32_t x, uint32_t y) {
    uint32_t lo, hi;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, 0, 0;" : "=r"(lo), "=r"(hi) : "r"(x), "r"(y));
    return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ fr_t mul_alu(const fr_t& a, const fr_t& b) {
    const uint32_t p[8] = {ZK_P0, ZK_P1, ZK_P2, ZK_P3, ZK_P4, ZK_P5, ZK_P6, ZK_P7};
    uint32_t t[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint32_t C = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint64_t uv = (uint64_t)a.v[j] * b.v[i] + add33(t[j], C);
            t[j] = (uint32_t)uv;
            C = (uint32_t)(uv >> 32);
        }
        t[8] += C;
        const uint32_t m = t[0] * 0xffffffffu;
        uint64_t C2 = (uint64_t)(t[0] != 0);
        {
            const uint64_t uv = ((uint64_t)m << 32) + t[1] + C2 - m;
            t[0] = (uint32_t)uv;
            C = (uint32_t)(uv >> 32);
        }
#pragma unroll
        for (int j = 2; j < 8; j++) {
            const uint64_t uv = (uint64_t)m * p[j] + add33(t[j], C);
            t[j - 1] = (uint32_t)uv;
            C = (uint32_t)(uv >> 32);
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

template <int V>
__device__ __forceinline__ fr_t MUL(const fr_t& a, const fr_t& b) {
    if (V == 0) return fr_mul(a, b);
    if (V == 1) return mul_u64(a, b);
    if (V == 3) return mul_u64p(a, b);
    if (V == 4) return mul_mix(a, b);
    if (V == 5) return mul_lazy(a, b);
    if (V == 8) return mul_alu(a, b);
    return mul_sos(a, b);
}

// Variant 6: three products per call through the production out-of-line fr_mul3_ni (k_relu_iround_f,
// k_sc_round2f); variant 7: one product per call (fr_mul_ni)
template <int V>
__global__ void __launch_bounds__(256) bench3(const fr_t* seed, uint32_t iters, fr_t* out) {
    uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    fr_t a = seed[tid & 1023], b = seed[(tid + 1) & 1023], c = seed[(tid + 2) & 1023];
    fr_t k = seed[(tid + 7) & 1023];
    for (uint32_t i = 0; i < iters; i++) {
        if (V == 6) {
            fr3_t r = fr_mul3_ni(a, k, b, k, c, k);
            a = r.x; b = r.y; c = r.z;
        } else {
            a = fr_mul_ni(a, k); b = fr_mul_ni(b, k); c = fr_mul_ni(c, k);
        }
    }
    out[tid] = fr_add(fr_add(a, b), c);
}

template <int V>
__global__ void __launch_bounds__(256) bench(const fr_t* seed, uint32_t iters, fr_t* out) {
    uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    fr_t a = seed[tid & 1023], b = seed[(tid + 1) & 1023], c = seed[(tid + 2) & 1023], d = seed[(tid + 3) & 1023];
    fr_t k = seed[(tid + 7) & 1023];
    for (uint32_t i = 0; i < iters; i++) {
        a = MUL<V>(a, k);
        b = MUL<V>(b, k);
        c = MUL<V>(c, k);
        d = MUL<V>(d, k);
    }
    out[tid] = fr_add(fr_add(a, b), fr_add(c, d));
}

template <int V>
__global__ void check(const fr_t* x, const fr_t* y, uint32_t n, int* bad) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        fr_t r0 = fr_mul(x[i], y[i]), r1 = MUL<V>(x[i], y[i]);
        if (V == 5) r1 = fr_reduce_once(r1);
        if (!fr_equal(r0, r1)) atomicAdd(bad, 1);
    }
}

static uint64_t rng = 88172645463325252ull;
static uint32_t next32() {
    rng ^= rng << 13;
    rng ^= rng >> 7;
    rng ^= rng << 17;
    return (uint32_t)rng;
}

template <int V>
static void run(const char* name, fr_t* d_seed, fr_t* d_out, int blocks, uint32_t iters) {
    int* bad;
    cudaMalloc(&bad, 4);
    cudaMemset(bad, 0, 4);
    check<V><<<64, 256>>>(d_seed, d_seed + 512, 512, bad);
    int hb = 0;
    cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    bench<V><<<blocks, 256>>>(d_seed, 10, d_out);
    float best = 1e30f;
    for (int r = 0; r < 3; r++) {
        cudaEventRecord(e0);
        bench<V><<<blocks, 256>>>(d_seed, iters, d_out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    double muls = (double)blocks * 256 * 4 * iters;
    cudaFuncAttributes at;
    cudaFuncGetAttributes(&at, bench<V>);
    printf("{\"variant\": \"%s\", \"blocks\": %d, \"G_frmul_per_s\": %.2f, \"regs\": %d, \"mismatches\": %d}\n", name, blocks,
           muls / (best / 1e3) / 1e9, at.numRegs, hb);
    cudaFree(bad);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); exit(1); }
}

template <int V>
static void run3(const char* name, fr_t* d_seed, fr_t* d_out, int blocks, uint32_t iters) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    bench3<V><<<blocks, 256>>>(d_seed, 10, d_out);
    float best = 1e30f;
    for (int r = 0; r < 3; r++) {
        cudaEventRecord(e0);
        bench3<V><<<blocks, 256>>>(d_seed, iters, d_out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFuncAttributes at;
    cudaFuncGetAttributes(&at, bench3<V>);
    printf("{\"variant\": \"%s\", \"blocks\": %d, \"G_frmul_per_s\": %.2f, \"regs\": %d}\n", name, blocks,
           (double)blocks * 256 * 3 * iters / (best / 1e3) / 1e9, at.numRegs);
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    // random canonical inputs (top limb < p7 keeps them < p) in Montgomery-agnostic form
    fr_t h[1024];
    for (int i = 0; i < 1024; i++) {
        for (int k = 0; k < 8; k++) h[i].v[k] = next32();
        h[i].v[7] &= 0x3fffffffu;
    }
    fr_t *d_seed, *d_out;
    cudaMalloc(&d_seed, sizeof h);
    cudaMemcpy(d_seed, h, sizeof h, cudaMemcpyHostToDevice);
    const int blocks = 148 * 8;
    cudaMalloc(&d_out, sizeof(fr_t) * blocks * 256);
    run<0>("ptx_cios", d_seed, d_out, blocks, 1000);
    run<1>("u64_cios", d_seed, d_out, blocks, 1000);
    run<3>("u64_cios_p01", d_seed, d_out, blocks, 1000);
    run<4>("mix_u64_madc", d_seed, d_out, blocks, 1000);
    run<5>("u64_p01_lazy", d_seed, d_out, blocks, 1000);
    run<8>("u64_p01_alucarry", d_seed, d_out, blocks, 1000);
    for (int b = 148 * 2; b <= 148 * 8; b *= 2) run3<6>("fr_mul3_ni", d_seed, d_out, b, 1000);
    for (int b = 148 * 2; b <= 148 * 8; b *= 2) run3<7>("fr_mul_ni x3", d_seed, d_out, b, 1000);
    return 0;
}
