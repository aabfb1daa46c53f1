// Latency of the device transcript step pieces on one warp (clock64 on lane 0), the first call cold and
// the steady state:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tr_bench scripts/tr_bench.cu
#include <cstdio>
#include "../paper_2307_16273_b200/csrc/transcript.cuh"
using namespace zk;

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__global__ void k_tr(uint8_t* st, long long* cyc, int iters) {
    __shared__ FsScratch fs;
    const int lane = threadIdx.x;
    fs_begin(fs, st);
    fr_t v = fr_from_u32(lane + 7);
    unsigned long long g0 = gtimer();
    long long c0 = clock64();
    for (int it = 0; it < iters; it++) {
        long long t0 = clock64();
        fs_absorb_frs(fs, "sc/msg", v, 3, nullptr);
        long long t1 = clock64();
        fr_t r = fs_challenge(fs, "sc/r");
        long long t2 = clock64();
        // pieces
        uint32_t h[8];
        hash_init(h);
        hash_compress(h, fs.buf[0], 64, true);
        long long t3 = clock64();
        fr_t c = fr_to_canonical_cold(r);
        long long t4 = clock64();
        fr_t c2 = fr_mul(r, v);
        long long t5 = clock64();
        fr_t c3 = fr_mul_f64(r, v);
        long long t6 = clock64();
        v = fr_add(v, fr_add(c, fr_add(c2, c3)));
        if (h[0] == 0x12345) v = fr_zero();
        if (lane == 0) {
            long long* o = cyc + 6 * it;
            o[0] = t1 - t0; o[1] = t2 - t1; o[2] = t3 - t2; o[3] = t4 - t3; o[4] = t5 - t4; o[5] = t6 - t5;
        }
        __syncwarp();
    }
    fs_end(fs, st);
    if (lane == 0) { cyc[6 * iters] = clock64() - c0; cyc[6 * iters + 1] = gtimer() - g0; }
}

// variant: MODE 1 = 256-thread block (warps 1-7 wait at __syncthreads), MODE 2 = + a large inlined
// integer-product loop between steps by all warps (instruction-cache pollution, as in k_sc_all)
template <int MODE>
__global__ void k_tr2(uint8_t* st, long long* cyc, int iters, const fr_t* src, fr_t* sink) {
    __shared__ FsScratch fs;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) fs_begin(fs, st);
    __syncthreads();
    fr_t v = fr_from_u32(lane + 7);
    for (int it = 0; it < iters; it++) {
        if (MODE == 2) {
            fr_t x = src[threadIdx.x], y = src[threadIdx.x + 1];
#pragma unroll
            for (int k = 0; k < 12; k++) x = fr_mul(fr_add(x, y), y);
            sink[threadIdx.x] = x;
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            long long t0 = clock64();
            fs_absorb_frs(fs, "sc/msg", v, 3, nullptr);
            long long t1 = clock64();
            fr_t r = fs_challenge(fs, "sc/r");
            long long t2 = clock64();
            v = fr_add(v, r);
            if (lane == 0) { cyc[2 * it] = t1 - t0; cyc[2 * it + 1] = t2 - t1; }
        }
        __syncthreads();
    }
    if (threadIdx.x < 32) fs_end(fs, st);
}

// variant: 33 blocks; block 0 runs the transcript steps and releases a flag per step, the other blocks
// wait for it with ld.volatile + nanosleep (the k_sc_all round structure without the products)
__global__ void k_tr3(uint8_t* st, long long* cyc, int iters, unsigned int* flag, uint8_t* proof) {
    __shared__ FsScratch fs;
    const int lane = threadIdx.x & 31;
    if (blockIdx.x == 0 && threadIdx.x < 32) fs_begin(fs, st);
    fr_t v = fr_from_u32(lane + 7);
    for (int it = 0; it < iters; it++) {
        if (blockIdx.x == 0) {
            if (threadIdx.x < 32) {
                long long t0 = clock64();
                fs_absorb_frs(fs, "sc/msg", v, 3, proof + 96 * it);
                long long t1 = clock64();
                fr_t r = fs_challenge(fs, "sc/r");
                long long t2 = clock64();
                v = fr_add(v, r);
                if (lane == 0) { cyc[2 * it] = t1 - t0; cyc[2 * it + 1] = t2 - t1; __threadfence(); atomicExch(flag, it + 1); }
            }
        } else if (threadIdx.x == 0) {
            unsigned int x;
            do { asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(x) : "l"(flag) : "memory"); if (x < (unsigned)it + 1) __nanosleep(256); } while (x < (unsigned)it + 1);
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) fs_end(fs, st);
}

int main() {
    uint8_t* st;
    long long* cyc;
    const int iters = 8;
    cudaMalloc(&st, 32);
    cudaMemset(st, 1, 32);
    cudaMallocManaged(&cyc, (6 * iters + 2) * sizeof(long long));
    k_tr<<<1, 32>>>(st, cyc, iters);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    const char* names[6] = {"absorb3", "challenge", "compress1", "canon_cold", "fr_mul_int", "fr_mul_f64"};
    for (int it = 0; it < iters; it++) {
        printf("iter %d:", it);
        for (int k = 0; k < 6; k++) printf(" %s %lld", names[k], cyc[6 * it + k]);
        printf("  (cycles)\n");
    }
    fr_t *src, *sink;
    cudaMalloc(&src, 512 * sizeof(fr_t));
    cudaMemset(src, 0, 512 * sizeof(fr_t));
    cudaMalloc(&sink, 512 * sizeof(fr_t));
    k_tr2<1><<<1, 256>>>(st, cyc, iters, src, sink);
    cudaDeviceSynchronize();
    printf("256-thread block: absorb3 %lld challenge %lld (iter 3)\n", cyc[6], cyc[7]);
    k_tr2<2><<<1, 256>>>(st, cyc, iters, src, sink);
    cudaDeviceSynchronize();
    printf("256-thread block + product loop between steps: absorb3 %lld challenge %lld (iter 3)\n", cyc[6], cyc[7]);
    unsigned int* flag;
    uint8_t* proof;
    cudaMalloc(&flag, 4);
    cudaMemset(flag, 0, 4);
    cudaMalloc(&proof, 96 * iters);
    k_tr3<<<33, 256>>>(st, cyc, iters, flag, proof);
    cudaDeviceSynchronize();
    printf("33 blocks, 32 waiting on a flag: absorb3 %lld challenge %lld (iter 3)\n", cyc[6], cyc[7]);
    cudaMemset(flag, 0, 4);
    k_tr3<<<1, 256>>>(st, cyc, iters, flag, proof);
    cudaDeviceSynchronize();
    printf("1 block (same code): absorb3 %lld challenge %lld (iter 3)\n", cyc[6], cyc[7]);
    cyc[6 * iters] = 0;
    k_tr<<<1, 32>>>(st, cyc, iters);
    cudaDeviceSynchronize();
    printf("total %lld cycles in %lld ns: %.3f GHz\n", cyc[6 * iters], cyc[6 * iters + 1], (double)cyc[6 * iters] / cyc[6 * iters + 1]);
    return 0;
}
