// common.cuh — runtime plumbing shared by the libzkdl translation units:
// context / transcript objects, error handling, launch accounting, grid-wide
// Fr reductions with a last-block finalizer, stream-ordered scratch memory.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>
#include <vector>

#include "../../include/zkdl.h"
#include "fr.cuh"
#include "transcript.cuh"

struct zk_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    int sm_budget = 0;         // cap on the grid of persistent kernels (0 = every SM), zk_ctx_set_sm_budget
    bool no_persist = false;   // zk_ctx_set_persistent(ctx, 0): per-round launches only
    void* nccl_comm = nullptr; // ncclComm_t owned by the context (zk_ctx_attach_nccl), sharded mode
    int nccl_rank = 0, nccl_world = 1;
    uint64_t launches = 0;
    std::string err;
    // a second stream for work off the critical path (created on first use; aux_ev: fork / join events)
    cudaStream_t aux = nullptr;
    cudaEvent_t aux_ev[2] = {nullptr, nullptr};
    cudaStream_t aux_stream() {
        if (!aux) {
            cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking);
            cudaEventCreateWithFlags(&aux_ev[0], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&aux_ev[1], cudaEventDisableTiming);
        }
        return aux;
    }
    // per-launch CUDA-event profiling (zk_ctx_profile): events bracket each launch on the ctx stream
    bool prof = false;
    std::string prof_filter;   // only this kernel, every template instantiation (empty: all kernels)
    bool prof_match(const char* name) const {
        if (!prof) return false;
        if (prof_filter.empty()) return true;
        const size_t n = prof_filter.size();
        return strncmp(name, prof_filter.c_str(), n) == 0 && (name[n] == '\0' || name[n] == '<');
    }
    struct Rec {
        const char* name;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> ev_pool;
    cudaEvent_t take_event() {
        if (!ev_pool.empty()) {
            cudaEvent_t e = ev_pool.back();
            ev_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
};

struct zk_transcript {
    zk_ctx* ctx = nullptr;
    uint8_t* d_st = nullptr;   // 32-byte transcript state (BLAKE2s digest, D3) on the device
};

namespace zk {

struct ZkError {
    zk_status st;
    std::string msg;
};

#define ZK_CUDA(call)                                                                                  \
    do {                                                                                               \
        cudaError_t e_ = (call);                                                                       \
        if (e_ != cudaSuccess)                                                                         \
            throw ::zk::ZkError{e_ == cudaErrorMemoryAllocation ? ZK_ERR_OOM : ZK_ERR_CUDA,            \
                                std::string(#call) + ": " + cudaGetErrorString(e_)};                   \
    } while (0)

#define ZK_REQUIRE(cond, status, text)                                                                 \
    do {                                                                                               \
        if (!(cond)) throw ::zk::ZkError{status, text};                                                \
    } while (0)

// Count and check a kernel launch (the launch count is reported by bench.py as gpu_launches).
inline void after_launch(zk_ctx* ctx, const char* what) {
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw ZkError{ZK_ERR_CUDA, std::string("launch ") + what + ": " + cudaGetErrorString(e)};
}
#define ZK_LAUNCH(ctx, kernel, grid, block, smem, ...)                                                 \
    do {                                                                                               \
        cudaEvent_t ev_a_ = nullptr, ev_b_ = nullptr;                                                  \
        const bool prof_ = (ctx)->prof_match(#kernel);                                                 \
        if (prof_) {                                                                                   \
            ev_a_ = (ctx)->take_event();                                                               \
            ev_b_ = (ctx)->take_event();                                                               \
            cudaEventRecord(ev_a_, (ctx)->stream);                                                     \
        }                                                                                              \
        kernel<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);                               \
        ::zk::after_launch((ctx), #kernel);                                                            \
        if (prof_) {                                                                                   \
            cudaEventRecord(ev_b_, (ctx)->stream);                                                     \
            (ctx)->recs.push_back({#kernel, ev_a_, ev_b_});                                            \
        }                                                                                              \
    } while (0)

// Stream-ordered scratch buffer (CUDA memory pool of the device), freed on scope exit.
struct Scratch {
    zk_ctx* ctx;
    std::vector<void*> ptrs;
    explicit Scratch(zk_ctx* c) : ctx(c) {}
    ~Scratch() {
        for (void* p : ptrs) cudaFreeAsync(p, ctx->stream);
    }
    template <typename T>
    T* alloc(size_t count) {
        void* p = nullptr;
        size_t bytes = count * sizeof(T);
        if (bytes == 0) bytes = 16;
        ZK_CUDA(cudaMallocAsync(&p, bytes, ctx->stream));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    template <typename T>
    T* alloc_zero(size_t count) {
        T* p = alloc<T>(count);
        ZK_CUDA(cudaMemsetAsync(p, 0, count * sizeof(T) ? count * sizeof(T) : 16, ctx->stream));
        return p;
    }
};

// ---------------------------------------------------------------- host-side field element helpers
// canonical check on the host (32-byte LE < p)
inline bool host_is_canonical(const uint8_t* b) {
    static const uint32_t P_[8] = {ZK_P0, ZK_P1, ZK_P2, ZK_P3, ZK_P4, ZK_P5, ZK_P6, ZK_P7};
    for (int i = 7; i >= 0; i--) {
        uint32_t w = (uint32_t)b[4 * i] | ((uint32_t)b[4 * i + 1] << 8) | ((uint32_t)b[4 * i + 2] << 16) |
                     ((uint32_t)b[4 * i + 3] << 24);
        if (w < P_[i]) return true;
        if (w > P_[i]) return false;
    }
    return false;   // equal to p
}
inline void check_canonical(const zk_fr* v, size_t n) {
    for (size_t i = 0; i < n; i++)
        ZK_REQUIRE(host_is_canonical(v[i].b), ZK_ERR_NONCANONICAL, "field element >= p");
}

// Upload n canonical host elements and convert to Montgomery form on the device.
void upload_points(zk_ctx* ctx, const zk_fr* host, uint32_t n, fr_t* d_mont, Scratch& s);

// ---------------------------------------------------------------- grid reduction with last-block finalize
// Every thread contributes acc[0..NV-1]; the block partials go to `partials` (gridDim.x * NV);
// the last block to arrive sums them and returns true on its thread 0 with the totals in out.
// `ticket` must be 0 on entry and is reset to 0 by the last block.  blockDim.x must be a multiple of 32.
template <int NV>
__device__ __forceinline__ void warp_reduce_fr(fr_t (&acc)[NV]) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int v = 0; v < NV; v++) acc[v] = fr_add(acc[v], fr_shfl_down(acc[v], off));
}

template <int NV>
__device__ __forceinline__ void block_reduce_fr(fr_t (&acc)[NV], fr_t* sm /* >= 32*NV */) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    warp_reduce_fr<NV>(acc);
    if (lane == 0)
#pragma unroll
        for (int v = 0; v < NV; v++) sm[wid * NV + v] = acc[v];
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int v = 0; v < NV; v++) acc[v] = lane < nw ? sm[lane * NV + v] : fr_zero();
        warp_reduce_fr<NV>(acc);
    }
    __syncthreads();
}

// The same with the shuffle levels rolled (~5x less code): for the persistent kernels' once-per-round
// reductions, whose code must stay in the instruction cache next to the transcript step.
template <int NV>
__device__ __forceinline__ void warp_reduce_fr_rolled(fr_t (&acc)[NV]) {
#pragma unroll 1
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int v = 0; v < NV; v++) acc[v] = fr_add(acc[v], fr_shfl_down(acc[v], off));
}
template <int NV>
__device__ __forceinline__ void block_reduce_fr_rolled(fr_t (&acc)[NV], fr_t* sm /* >= 32*NV */) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    warp_reduce_fr_rolled<NV>(acc);
    if (lane == 0)
#pragma unroll
        for (int v = 0; v < NV; v++) sm[wid * NV + v] = acc[v];
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int v = 0; v < NV; v++) acc[v] = lane < nw ? sm[lane * NV + v] : fr_zero();
        warp_reduce_fr_rolled<NV>(acc);
    }
    __syncthreads();
}

template <int NV>
__device__ bool grid_reduce_fr(fr_t (&acc)[NV], fr_t* partials, unsigned int* ticket, fr_t (&out)[NV]) {
    __shared__ fr_t sm[32 * NV];
    __shared__ bool is_last;
    block_reduce_fr<NV>(acc, sm);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int v = 0; v < NV; v++) fr_store(&partials[blockIdx.x * NV + v], acc[v]);
        __threadfence();
        unsigned int t = atomicAdd(ticket, 1u);
        is_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!is_last) return false;
    __threadfence();
    fr_t s[NV];
#pragma unroll
    for (int v = 0; v < NV; v++) s[v] = fr_zero();
    for (unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x)
#pragma unroll
        for (int v = 0; v < NV; v++) {
            const uint4* q = reinterpret_cast<const uint4*>(&partials[b * NV + v]);
            uint4 x = __ldcg(q), y = __ldcg(q + 1);
            s[v] = fr_add(s[v], fr_t{{x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w}});
        }
    block_reduce_fr<NV>(s, sm);
    if (threadIdx.x == 0) {
        *ticket = 0;
#pragma unroll
        for (int v = 0; v < NV; v++) out[v] = s[v];
        return true;
    }
    return false;
}

// Same as grid_reduce_fr but returns true on EVERY thread of the last block; the totals are in
// `out_sm` (shared, NV entries) after the call (so the whole last block can run a finalize step).
template <int NV>
__device__ bool grid_reduce_fr_block(fr_t (&acc)[NV], fr_t* partials, unsigned int* ticket, fr_t* out_sm) {
    __shared__ fr_t sm[32 * NV];
    __shared__ bool is_last;
    block_reduce_fr<NV>(acc, sm);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int v = 0; v < NV; v++) fr_store(&partials[blockIdx.x * NV + v], acc[v]);
        __threadfence();
        unsigned int t = atomicAdd(ticket, 1u);
        is_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!is_last) return false;
    __threadfence();
    fr_t s[NV];
#pragma unroll
    for (int v = 0; v < NV; v++) s[v] = fr_zero();
    for (unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x)
#pragma unroll
        for (int v = 0; v < NV; v++) {
            const uint4* q = reinterpret_cast<const uint4*>(&partials[b * NV + v]);
            uint4 x = __ldcg(q), y = __ldcg(q + 1);
            s[v] = fr_add(s[v], fr_t{{x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w}});
        }
    block_reduce_fr<NV>(s, sm);
    if (threadIdx.x == 0) {
        *ticket = 0;
#pragma unroll
        for (int v = 0; v < NV; v++) out_sm[v] = s[v];
    }
    __syncthreads();
    return true;
}

inline unsigned int grid_for(zk_ctx* ctx, uint64_t work_items, int threads, int blocks_per_sm = 4) {
    uint64_t need = (work_items + threads - 1) / threads;
    uint64_t cap = (uint64_t)ctx->num_sms * blocks_per_sm;
    if (need < 1) need = 1;
    return (unsigned int)(need < cap ? need : cap);
}

// Small fixed-capacity byte string passed to kernels by value (tags, headers).
struct Bytes256 {
    uint32_t len;
    uint8_t b[256];
};
inline Bytes256 make_bytes(const void* p, size_t n) {
    ZK_REQUIRE(n <= 256, ZK_ERR_ARG, "message too long for by-value transfer");
    Bytes256 r;
    r.len = (uint32_t)n;
    if (n) memcpy(r.b, p, n);
    return r;
}
struct Tag32 {
    char s[32];
};
inline Tag32 make_tag(const char* t) {
    size_t n = strlen(t);
    ZK_REQUIRE(n < 32, ZK_ERR_ARG, "tag longer than 31 bytes");
    Tag32 r;
    memset(r.s, 0, sizeof r.s);
    memcpy(r.s, t, n);
    return r;
}

// ---------------------------------------------------------------- shared kernels (defined in transcript.cu)
__global__ void k_tr_absorb(uint8_t* st, Tag32 tag, Bytes256 msg, uint8_t* copy_out);
__global__ void k_tr_absorb_dev(uint8_t* st, Tag32 tag, const uint8_t* msg, uint64_t len);
__global__ void k_tr_absorb_frs(uint8_t* st, Tag32 tag, const fr_t* v, uint32_t n, uint8_t* copy_out);
// n challenges with one tag: thread 0 advances the state chain, all threads squeeze in parallel.
__global__ void k_tr_challenges(uint8_t* st, Tag32 tag, uint32_t n, fr_t* out_mont, uint8_t* out_canon);

// Host wrappers
// d_copy (nullable, len <= 256 only): the kernel also writes msg to this device buffer
void tr_absorb_host(zk_transcript* tr, const char* tag, const void* msg, size_t len, uint8_t* d_copy = nullptr);
void tr_challenges_dev(zk_transcript* tr, const char* tag, uint32_t n, fr_t* d_out_mont, uint8_t* d_out_canon);
// k <= 4 challenge vectors (tags[t], ns[t] each, Montgomery outputs) drawn in order in one launch: the same
// transcript as k tr_challenges_dev calls
void tr_challenges_multi_dev(zk_transcript* tr, uint32_t k, const char* const* tags, const uint32_t* ns,
                             fr_t* const* d_out_mont, uint8_t* const* d_out_canon = nullptr);

// eq tables (tables.cu): out[x] = scale * prod_{s<k} eq(u[s], bit s of x) for x < 2^k
void eq_table_dev(zk_ctx* ctx, const fr_t* d_u, uint32_t k, const fr_t* d_scale, fr_t* d_out, Scratch& s);
// Montgomery <-> canonical conversion of device tables
void to_canonical_dev(zk_ctx* ctx, const fr_t* in, uint64_t n, uint8_t* out);

}  // namespace zk
