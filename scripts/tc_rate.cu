// tcgen05.mma kind::i8 issue-rate probe: each CTA (one per SM) issues `iters` groups of `per` MMAs
// (M = 128, K = 32, N = n) with A in TMEM (or, SS, in shared memory) and B in shared memory, accumulating into `per` separate
// accumulators, then commits once.  Prints Tera-MAC/s per N.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tc_rate scripts/tc_rate.cu && ./tc_rate
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int N, bool SS>
__global__ void rate(int iters, int per, int* sink) {
    __shared__ __align__(1024) uint8_t sB[256 * 32];
    __shared__ __align__(1024) uint8_t sA[4 * 4096];   // SS: A tiles in shared memory
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (int)sizeof(sB); i += blockDim.x) sB[i] = (uint8_t)(i & 1);
    for (int i = threadIdx.x; i < (int)sizeof(sA); i += blockDim.x) sA[i] = (uint8_t)(i & 3);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tmem_base;
    const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t bd = (uint64_t)((su32(sB) >> 4) & 0x3fff) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
                        (1ull << 46);
    if (threadIdx.x == 0) {
        const uint32_t acol = 480;   // A tile at columns [480, 488)
        for (int it = 0; it < iters; it++)
            for (int p = 0; p < per; p++) {
                const uint32_t d = tb + (uint32_t)((p * N) % 448);
                if (SS) {
                    const uint64_t ad = (uint64_t)((su32(sA + 4096 * (p & 3)) >> 4) & 0x3fff) | ((uint64_t)(128 >> 4) << 16) |
                                        ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
                    asm volatile(
                        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, q;\n\t}" ::"r"(d),
                        "l"(ad), "l"(bd), "r"(idesc), "r"(it));
                    continue;
                }
                asm volatile(
                    "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, q;\n\t}" ::"r"(d),
                    "r"(tb + acol), "l"(bd), "r"(idesc), "r"(it));
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar)));
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(su32(&mbar)));
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
    if (threadIdx.x == 0) sink[blockIdx.x] = 1;
}

template <int N, bool SS = false>
void run(int per, int* sink) {
    const int iters = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    rate<N, SS><<<148, 128>>>(10, per, sink);
    cudaEventRecord(a);
    rate<N, SS><<<148, 128>>>(iters, per, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double macs = 148.0 * iters * per * 128.0 * N * 32.0;
    printf("{\"ss\": %d, \"N\": %d, \"per\": %d, \"ns_per_mma\": %.2f, \"TMAC_s\": %.1f, \"err\": \"%s\"}\n", (int)SS, N,
           per, ms * 1e6 / ((double)iters * per), macs / (ms / 1e3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int* sink;
    cudaMalloc(&sink, 4096);
    run<32>(9, sink);
    run<32>(1, sink);
    run<64>(5, sink);
    run<128>(3, sink);
    run<256>(1, sink);
    run<32, true>(9, sink);
    run<32, true>(4, sink);
    run<64, true>(4, sink);
    run<96, true>(4, sink);
    run<128, true>(3, sink);
    run<256, true>(1, sink);
    return 0;
}
