// Fr product on the FP64 pipe (csrc/fr64.cuh) against the integer CIOS (csrc/fr.cuh): bit-exactness on
// random and edge inputs, and register-resident throughput (G Fr-mul/s) for 1-4 independent chains per
// thread, alone and interleaved with the integer product (do the two pipes add?).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/fr64_bench scripts/fr64_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../paper_2307_16273_b200/csrc/fr.cuh"

using namespace zk;

__device__ uint64_t splitmix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ fr_t rnd(uint64_t s, bool below_p) {
    fr_t x;
    for (int i = 0; i < 4; i++) {
        uint64_t r = splitmix(s * 8 + i);
        x.v[2 * i] = (uint32_t)r;
        x.v[2 * i + 1] = (uint32_t)(r >> 32);
    }
    if (below_p) {
        x.v[7] &= 0x3fffffffu;   // < 2^254 < p
    }
    return x;
}

__global__ void k_check(uint64_t n, unsigned long long* bad, fr_t* first_bad) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
        fr_t a = rnd(2 * t, true), b = rnd(2 * t + 1, (t & 1) != 0);
        const int e = (int)(t % 97);
        if (e == 0) a = fr_const(ZK_P0 - 1 + 0, ZK_P1, ZK_P2, ZK_P3, ZK_P4, ZK_P5, ZK_P6, ZK_P7);   // p - 1 (p0 = 1)
        if (e == 1) b = fr_const(~0u, ~0u, ~0u, ~0u, ~0u, ~0u, ~0u, ~0u);                          // 2^256 - 1
        if (e == 2) a = fr_zero();
        if (e == 3) { a = fr_const(ZK_P0 - 1, ZK_P1, ZK_P2, ZK_P3, ZK_P4, ZK_P5, ZK_P6, ZK_P7); b = fr_const(~0u, ~0u, ~0u, ~0u, ~0u, ~0u, ~0u, ~0u); }
        if (e == 4) { a.v[0] = 1; for (int i = 1; i < 8; i++) a.v[i] = 0; }
        const fr_t x = fr_mul(a, b), y = fr_mul_f64(a, b), z = fr_mul_f64r(a, b);
        if (!fr_equal(x, y) || !fr_equal(x, z)) {
            if (atomicAdd(bad, 1ull) == 0) { first_bad[0] = a; first_bad[1] = b; first_bad[2] = x; first_bad[3] = y; }
        }
    }
}

template <int C, int MODE>   // MODE 0: integer CIOS, 1: FP64, 2: half the chains each, 3: odd warps integer, even warps FP64,
                             // 4: FP64 rolled (CIOS order)
__global__ void __launch_bounds__(256) k_rate(const fr_t* seed, uint32_t iters, fr_t* out) {
    fr_t x[C];
    const fr_t y = seed[(threadIdx.x + 1) & 1023];
#pragma unroll
    for (int c = 0; c < C; c++) x[c] = seed[(threadIdx.x * C + c) & 1023];
    for (uint32_t i = 0; i < iters; i++) {
#pragma unroll
        for (int c = 0; c < C; c++) {
            if (MODE == 4) x[c] = fr_mul_f64r(x[c], y);
            else if (MODE == 0 || (MODE == 2 && (c & 1)) || (MODE == 3 && ((threadIdx.x >> 5) & 1))) x[c] = fr_mul(x[c], y);
            else x[c] = fr_mul_f64(x[c], y);
        }
    }
    fr_t acc = x[0];
#pragma unroll
    for (int c = 1; c < C; c++) acc = fr_add(acc, x[c]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int C, int MODE>
void rate(const char* name, const fr_t* seed, fr_t* out, int bps) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rate<C, MODE>, 256, 0);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_rate<C, MODE>);
    const int blocks = 148 * (bps ? bps : per_sm);
    const uint32_t iters = 2048 / C;
    k_rate<C, MODE><<<blocks, 256>>>(seed, 4, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_rate<C, MODE><<<blocks, 256>>>(seed, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double n = (double)blocks * 256 * iters * C;
    printf("{\"variant\": \"%s\", \"chains\": %d, \"blocks_per_sm\": %d, \"regs\": %d, \"G_frmul_per_s\": %.2f}\n", name, C,
           blocks / 148, fa.numRegs, n / (ms / 1e3) / 1e9);
}

int main() {
    unsigned long long* bad;
    fr_t* fb;
    cudaMallocManaged(&bad, 8);
    cudaMallocManaged(&fb, 4 * sizeof(fr_t));
    *bad = 0;
    const uint64_t n = 1ull << 26;
    k_check<<<148 * 8, 256>>>(n, bad, fb);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
    printf("{\"check\": %llu, \"mismatches\": %llu}\n", (unsigned long long)n, *bad);
    if (*bad) {
        for (int k = 0; k < 4; k++) {
            printf("  ");
            for (int i = 7; i >= 0; i--) printf("%08x", fb[k].v[i]);
            printf("\n");
        }
    }
    fr_t *seed, *out;
    cudaMalloc(&seed, 1024 * sizeof(fr_t));
    cudaMalloc(&out, 148 * 32 * 256 * sizeof(fr_t));
    fr_t hs[1024];
    for (int i = 0; i < 1024; i++)
        for (int l = 0; l < 8; l++) hs[i].v[l] = (uint32_t)(0x9E3779B9u * (i * 8 + l + 1)) & (l == 7 ? 0x3fffffffu : ~0u);
    cudaMemcpy(seed, hs, sizeof hs, cudaMemcpyHostToDevice);
    rate<4, 0>("int_cios", seed, out, 0);
    rate<1, 1>("fp64", seed, out, 0);
    rate<2, 1>("fp64", seed, out, 0);
    rate<4, 1>("fp64", seed, out, 0);
    rate<2, 2>("mixed", seed, out, 0);
    rate<4, 2>("mixed", seed, out, 0);
    for (int bps : {1, 2, 3, 4}) rate<2, 1>("fp64", seed, out, bps);
    rate<1, 4>("fp64_rolled", seed, out, 0);
    rate<2, 4>("fp64_rolled", seed, out, 0);
    rate<1, 3>("per_warp_mixed", seed, out, 0);
    rate<2, 3>("per_warp_mixed", seed, out, 0);
    rate<3, 3>("per_warp_mixed", seed, out, 0);
    rate<3, 1>("fp64", seed, out, 0);
    rate<3, 0>("int_cios", seed, out, 0);
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
    return 0;
}
