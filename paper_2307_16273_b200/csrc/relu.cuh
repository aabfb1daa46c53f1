// relu.cuh — zkReLU tables and aggregated six-statement sumcheck (rows a7, a8).
#pragma once
#include "common.cuh"

namespace zk {

struct ReluOutputs {
    uint8_t* d_proof;   // relu_proof_len bytes
    uint8_t* d_point;   // (logB + logD) canonical challenges
};

inline uint32_t relu_logB(uint32_t Q, uint32_t R) {
    uint32_t qr = Q + R, l = 0;
    while ((1u << l) < qr) l++;
    return l;
}
inline uint64_t relu_proof_len(uint32_t logD, uint32_t logB) { return 12 + 128 + 128ull * (logB + logD) + 96; }

bool relu_tables_dev(zk_ctx* ctx, const int32_t* Z, const int32_t* GA, uint64_t D, uint32_t Q, uint32_t R, uint8_t* sign,
                     int32_t* A, int32_t* GZ, int32_t* Zp, int32_t* GAp, int32_t* RZ, int32_t* RGA, Scratch& s);

// Bit-sum cells on the tensor cores (gram.cu): writes the 4B + B(B+1) cell totals in cell_decode order, and
// lin6[s][par][q][j] (12 B values): the linear cells per parity of the first i-variable over pairs b,
// sum_b eq(u_x[1..], b) g_q(b) bit_j(w_s(2b + par)) (g_0 = 1, g_1 = o(2b + par), g_2 = o(2b + 1 - par), o = 1 - sig;
// x = 2s for q = 0, 2s + 1 otherwise), from which the first i-round's linear terms follow.
bool relu_gram_supported(uint32_t logD, uint32_t B);
void relu_bitsums_gram(zk_ctx* ctx, const int32_t* Z, const int32_t* GA, uint32_t logD, uint32_t qr_mask,
                       uint32_t sig_bit, uint32_t B, const fr_t* const u_i[5], fr_t* cell_tot, fr_t* lin6, Scratch& s);

// Enqueues the whole proof; bit 0 of *range_flag (device word, not cleared here) is set if an input
// lies outside the (Q+R)-bit range (never for Q+R = 32: every int32 is in range).
void relu_prove_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* Z, const int32_t* GA, uint32_t logD, uint32_t Q,
                    uint32_t R, ReluOutputs& out, unsigned int* range_flag, Scratch& s,
                    const uint8_t* d_pts = nullptr /* chained (D25): 4 x logD canonical points, device */);

}  // namespace zk
