// Do cooperative launches on different streams run concurrently?  Two spin kernels (each `ns` long, G CTAs)
// on two streams, launched (a) with cudaLaunchCooperativeKernel, (b) as plain launches; prints the elapsed
// time of each pair (concurrent ~ ns, serialised ~ 2 ns).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(unsigned long long ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < ns);
}
int main() {
    cudaStream_t s[4];
    for (int i = 0; i < 4; i++) cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    unsigned long long ns = 200000;
    void* args[] = {&ns};
    for (int G : {8, 37, 74}) for (int coop = 0; coop < 2; coop++) for (int nstr : {1, 2, 4}) {
        float best = 1e9;
        for (int rep = 0; rep < 5; rep++) {
            cudaDeviceSynchronize();
            cudaEventRecord(a, s[0]);
            for (int i = 1; i < nstr; i++) cudaStreamWaitEvent(s[i], a, 0);
            for (int i = 0; i < nstr; i++) {
                if (coop) cudaLaunchCooperativeKernel((void*)spin, dim3(G), dim3(256), args, 0, s[i]);
                else spin<<<G, 256, 0, s[i]>>>(ns);
            }
            cudaEvent_t e[4];
            for (int i = 1; i < nstr; i++) { cudaEventCreate(&e[i]); cudaEventRecord(e[i], s[i]); cudaStreamWaitEvent(s[0], e[i], 0); }
            cudaEventRecord(b, s[0]);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("G=%3d %-11s streams=%d: %.3f ms (one kernel 0.200)\n", G, coop ? "cooperative" : "plain", nstr, best);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
