// tcgen05 kind::i8 probe for an MN-major A operand (the column-sum contraction out[c] = sum_r M[r][c] E(r)):
// D[128 x 32] (s32, TMEM) = A^T B^T with A[k][m] = bytes of K = 32 matrix rows x 128 bytes (M = 128 byte
// columns), stored as the TMA SWIZZLE_128B box would (row k at 128 k, 16-byte chunk j at chunk j ^ (k % 8)),
// instruction descriptor a_major = 1 (bit 15), smem descriptor layout SW128 with SBO = 1024 B; B[n][k]
// K-major, no swizzle.  Checks u8 and s8 A against a CPU product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tc_mn_probe scripts/tc_mn_probe.cu && ./tc_mn_probe
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 32, K = 32;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const uint8_t* A, const uint8_t* B, int32_t* D, uint32_t idesc, uint32_t lbo, uint32_t sbo) {
    __shared__ __align__(1024) uint8_t sA[K * M];
    __shared__ __align__(1024) uint8_t sB[N * K];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    for (int e = threadIdx.x; e < K * M; e += blockDim.x) {   // SW128: row k, chunk j -> chunk j ^ (k & 7)
        const int k = e / M, m = e % M, j = m / 16;
        sA[k * 128 + ((j ^ (k & 7)) * 16) + (m % 16)] = A[k * M + m];
    }
    for (int e = threadIdx.x; e < N * K; e += blockDim.x) {   // K-major no swizzle
        const int n = e / K, kb = e % K;
        sB[(n / 8) * 256 + (kb / 16) * 128 + (n % 8) * 16 + (kb % 16)] = B[n * K + kb];
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tmem_base;
    if (threadIdx.x == 0) {
        const uint64_t ad = (uint64_t)((su32(sA) >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
                            ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46) | (2ull << 61);
        const uint64_t bd = (uint64_t)((su32(sB) >> 4) & 0x3fff) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
                            (1ull << 46);
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, q;\n\t}" ::"r"(tb),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar)));
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done) : "r"(su32(&mbar)));
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp < 4) {
        uint32_t v[32];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
                     "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
                       "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
                       "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
                       "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                     : "r"(tb + ((32 * warp) << 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int n = 0; n < 32; n++) D[(32 * warp + lane) * N + n] = (int32_t)v[n];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tb));
}

int main() {
    std::vector<uint8_t> A(K * M), B(N * K);
    srand(7);
    for (auto& x : A) x = rand() & 255;
    for (auto& x : B) x = rand() & 255;
    uint8_t *dA, *dB;
    int32_t* dD;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, B.size());
    cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    for (int sgn = 0; sgn < 2; sgn++)
        for (uint32_t lbo : {16u, 128u, 1024u}) {
            const uint32_t idesc = (2u << 4) | ((uint32_t)sgn << 7) | (1u << 15) | ((N >> 3) << 17) | ((M >> 4) << 24);
            cudaMemset(dD, 0, M * N * 4);
            probe<<<1, 128>>>(dA, dB, dD, idesc, lbo, 1024);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<int32_t> D(M * N);
            cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int m = 0; m < M; m++)
                for (int n = 0; n < N; n++) {
                    int64_t ref = 0;
                    for (int k = 0; k < K; k++) ref += (int64_t)(sgn ? (int8_t)A[k * M + m] : A[k * M + m]) * B[n * K + k];
                    if (ref != D[m * N + n]) bad++;
                }
            printf("a_major=MN sw128 %s lbo=%u: %s, %d / %d mismatches (D[0][0]=%d)\n", sgn ? "s8" : "u8", lbo,
                   cudaGetErrorString(e), bad, M * N, D[0]);
        }
    return 0;
}
