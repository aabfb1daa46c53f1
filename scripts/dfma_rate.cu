// FP64 FMA vs 32-bit IMAD issue rates on this GPU (is an FP64-limb Montgomery product worth it?).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_rate scripts/dfma_rate.cu && ./dfma_rate
#include <cstdint>
#include <cstdio>

__global__ void dfma_k(double* out, int iters, double s) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int i = 0; i < iters; i++) {
        a0 = fma(a0, s, 1.0); a1 = fma(a1, s, 1.0); a2 = fma(a2, s, 1.0); a3 = fma(a3, s, 1.0);
        a4 = fma(a4, s, 1.0); a5 = fma(a5, s, 1.0); a6 = fma(a6, s, 1.0); a7 = fma(a7, s, 1.0);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void imad_k(uint32_t* out, int iters, uint32_t s) {
    uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int i = 0; i < iters; i++) {
        a0 = a0 * s + 1; a1 = a1 * s + 1; a2 = a2 * s + 1; a3 = a3 * s + 1;
        a4 = a4 * s + 1; a5 = a5 * s + 1; a6 = a6 * s + 1; a7 = a7 * s + 1;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void imadw_k(uint64_t* out, int iters, uint32_t s) {
    uint64_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    uint32_t b0 = threadIdx.x, b1 = b0 + 1, b2 = b0 + 2, b3 = b0 + 3;
    for (int i = 0; i < iters; i++) {   // IMAD.WIDE.U32: 32x32 + 64 -> 64
        a0 = (uint64_t)b0 * s + a0; a1 = (uint64_t)b1 * s + a1; a2 = (uint64_t)b2 * s + a2; a3 = (uint64_t)b3 * s + a3;
        b0 = (uint32_t)a0; b1 = (uint32_t)a1; b2 = (uint32_t)a2; b3 = (uint32_t)a3;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}

template <class K, class T, class S>
void run(const char* name, K k, T* out, S s, int ops_per_iter) {
    const int blocks = 148 * 8, threads = 256, iters = 4096;
    k<<<blocks, threads>>>(out, 16, s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<blocks, threads>>>(out, iters, s);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = (double)blocks * threads * iters * ops_per_iter;
    printf("{\"op\": \"%s\", \"T_per_s\": %.2f, \"per_sm_per_clk_at_1965\": %.1f}\n", name, ops / (ms / 1e3) / 1e12,
           ops / (ms / 1e3) / 148 / 1.965e9);
}

int main() {
    double* d;
    uint32_t* u;
    uint64_t* w;
    cudaMalloc(&d, 148 * 8 * 256 * 8);
    cudaMalloc(&u, 148 * 8 * 256 * 4);
    cudaMalloc(&w, 148 * 8 * 256 * 8);
    run("DFMA", dfma_k, d, 0.999, 8);
    run("IMAD", imad_k, u, 3u, 8);
    run("IMAD.WIDE", imadw_k, w, 3u, 4);
    return 0;
}
