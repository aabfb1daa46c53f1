// sumcheck.cuh — device-side product sumcheck driver interface (rows a4-a6).
#pragma once
#include "common.cuh"

namespace zk {

struct ScStatement {
    uint32_t m, n_eq, K;
    const fr_t* tables[3];   // Fr (Montgomery), 2^m entries each; not modified
    const fr_t* d_w;         // n_eq points (Montgomery)
    fr_t* d_claim;           // in (claim_given) or out
    bool claim_given;
    uint8_t* d_proof;        // sumcheck_proof_len(m, K) bytes
    fr_t* d_r;               // m challenges (Montgomery)
    uint8_t* d_point;        // m challenges (canonical)
    fr_t* d_finals;          // K finals (Montgomery), may be null
};

void sumcheck_prove_dev(zk_ctx* ctx, zk_transcript* tr, const ScStatement& S, Scratch& s);
uint64_t sumcheck_proof_len(uint32_t m, uint32_t K);

}  // namespace zk
