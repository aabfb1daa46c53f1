// tcgen05 kind::i8 probe: D[128 x N] (s32, TMEM) = A[128 x K] (u8, TMEM) * B[N x K]^T (u8, SMEM, K-major,
// no swizzle), K = 32 * ksteps.  Validates the operand layouts and descriptors used by the zkReLU
// bit-sum kernel against a CPU product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tc_probe scripts/tc_probe.cu && ./tc_probe
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

constexpr int M = 128, N = 32, KSTEPS = 4, K = 32 * KSTEPS;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_kmajor_noswizzle(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}

__global__ void probe(const uint8_t* A, const uint8_t* B, int32_t* D, uint32_t idesc) {
    __shared__ __align__(1024) uint8_t sB[KSTEPS][N * 32];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    // B tile per k-step: row n (0..N-1), K bytes 0..31: 8-row groups of 256 B = [k 0..15 x 8 rows][k 16..31 x 8 rows]
    for (int e = threadIdx.x; e < KSTEPS * N * 32; e += blockDim.x) {
        int ks = e / (N * 32), r = e % (N * 32), n = r / 32, kb = r % 32;
        int off = (n / 8) * 256 + (kb / 16) * 128 + (n % 8) * 16 + (kb % 16);
        sB[ks][off] = B[n * K + ks * 32 + kb];
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tmem_base;
    // A into TMEM columns [N, N + 8*KSTEPS): row m = lane 32*warp + lane, k-step ks at columns N + 8 ks
    if (warp < 4) {
        const int m = 32 * warp + lane;
        for (int ks = 0; ks < KSTEPS; ks++) {
            uint32_t w[8];
            for (int c = 0; c < 8; c++) {
                const uint8_t* p = A + m * K + ks * 32 + 4 * c;
                w[c] = p[0] | (p[1] << 8) | (p[2] << 16) | ((uint32_t)p[3] << 24);
            }
            const uint32_t ta = tb + ((uint32_t)(32 * warp) << 16) + N + 8 * ks;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(ta), "r"(w[0]),
                         "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        for (int ks = 0; ks < KSTEPS; ks++) {
            const uint64_t bd = desc_kmajor_noswizzle(smem_u32(sB[ks]), 128, 256);
            const uint32_t ta = tb + N + 8 * ks;
            const uint32_t acc = ks > 0;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tb),
                "r"(ta), "l"(bd), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
    }
    // wait for the MMAs
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(smem_u32(&mbar)), "r"(0));
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp < 4) {
        uint32_t v[32];
        const uint32_t ta = tb + ((uint32_t)(32 * warp) << 16);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
            "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
              "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
              "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
              "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        const int m = 32 * warp + lane;
        for (int n = 0; n < N; n++) D[m * N + n] = (int32_t)v[n];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(256));
}

int main() {
    std::vector<uint8_t> A(M * K), B(N * K);
    srand(7);
    for (auto& x : A) x = rand() & 255;
    for (auto& x : B) x = rand() & 1;
    uint8_t *dA, *dB;
    int32_t* dD;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, B.size());
    cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    cudaMemset(dD, 0xff, M * N * 4);
    // kind::i8 instruction descriptor: D s32 (bits 4-5 = 2), A/B u8 (0), K-major, N >> 3 at bit 17, M >> 4 at bit 24
    const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    probe<<<1, 160>>>(dA, dB, dD, idesc);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<int32_t> D(M * N);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < M; m++)
        for (int n = 0; n < N; n++) {
            int32_t ref = 0;
            for (int k = 0; k < K; k++) ref += A[m * K + k] * B[n * K + k];
            if (ref != D[m * N + n]) {
                if (bad < 8) printf("mismatch m=%d n=%d got %d want %d\n", m, n, D[m * N + n], ref);
                bad++;
            }
        }
    printf("{\"tc_probe\": \"%s\", \"mismatches\": %d}\n", bad ? "FAIL" : "ok", bad);
    return bad != 0;
}
