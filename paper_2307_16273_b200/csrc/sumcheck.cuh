// sumcheck.cuh — device-side product sumcheck driver interface (rows a4-a6, §8(e) sharding).
#pragma once
#include "common.cuh"

namespace zk {

struct ScStatement {
    uint32_t m, n_eq, K;
    const fr_t* tables[3];   // Fr (Montgomery), 2^m entries each; not modified (i32[k] set: scratch that
                             // round 0 fills with the embedded int32 table)
    const int32_t* i32[3];   // int32 source of table k, or null
    const fr_t* d_w;         // n_eq points (Montgomery)
    fr_t* d_claim;           // in (claim_given) or out
    bool claim_given;
    uint8_t* d_proof;        // sumcheck_proof_len(m, K) bytes
    fr_t* d_r;               // m challenges (Montgomery)
    uint8_t* d_point;        // m challenges (canonical)
    fr_t* d_finals;          // K finals (Montgomery), may be null
};

// Round engine shared by the single-device prover, the sharded prover (partial + combine per round)
// and the continuation after the sharded tables are gathered onto every rank.
struct ScEngine {
    zk_ctx* ctx = nullptr;
    zk_transcript* tr = nullptr;
    Scratch* s = nullptr;
    uint32_t m = 0, n_eq = 0, K = 0;   // global statement
    uint32_t L = 0, t0 = 0, n_eq_loc = 0, t = 0;
    const fr_t* cur[3] = {nullptr, nullptr, nullptr};
    fr_t* buf[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
    fr_t *HI = nullptr, *LO[2] = {nullptr, nullptr}, *HP[2] = {nullptr, nullptr};
    uint32_t hb = 0, lo0 = 0;
    int lo_level = 0, hp_next = 0;
    const fr_t* hi_cur = nullptr;
    const fr_t* d_w = nullptr;
    const fr_t* d_scale = nullptr;
    fr_t* partials = nullptr;
    unsigned int* ticket = nullptr;
    uint8_t* d_proof = nullptr;
    fr_t* d_r = nullptr;
    uint8_t* d_point = nullptr;
    fr_t* d_claim = nullptr;
    bool claim_given = false;
    fr_t* d_finals = nullptr;
    const int32_t* i32[3] = {nullptr, nullptr, nullptr};   // int32 sources: round 0 embeds into cur[k]
    bool factored = true;   // K = 2: k_sc_round2f (ZKDL_SC_V=0: the unfactored k_sc_round)
    bool zero = false;      // N2 zero form (D22): K = 3 tables (Y, A, B), terms Y - A B, 3 evaluations
    bool int0_used = false; // round 0 ran on the int32 tables in integers (cur[] not embedded; round 1 folds
                            // from the int32 tables)
    // derived X = 1 (single-device provers from round 0, K = 2 factored): the running claim every
    // finalizer updates and w_t^-1 (computed on the aux stream; the rounds from 1 on wait for it)
    bool derive = false;
    fr_t* run_claim = nullptr;
    fr_t* winv = nullptr;
    uint32_t nev() const { return zero ? 3 : K + 1; }   // evaluations per round message

    // int32 tables: round 0 of the factored kernel embeds them into the (scratch) cur tables; otherwise
    // they are embedded here, before round 0
    void set_i32(const int32_t* const src[3]);
    // make cur[] hold the Fr tables the next round expects (embeds int32 tables round 0 left in
    // integers); for consumers other than round(): persist_rest, the shard export
    void materialize();
    // local tables of 2^L entries entering at global round t0; eq over w[t0 .. t0 + n_eq_loc - 1]
    void setup(const fr_t* const tables[3], uint32_t L, uint32_t t0, uint32_t n_eq_loc);
    void header();                    // absorb "sc/hdr" (+ the given claim)
    void round(fr_t* part_out);       // round t: fused (part_out == nullptr) or partial-only
    void combine(const fr_t* all, uint32_t G);   // sharded: sum G partials + transcript step of round t-1
    void finals();
    // every remaining round and the finals; the last rounds (<= 2^SC_TAIL_LOG entries left) in one
    // persistent cooperative launch instead of one launch per round
    void run_to_end();
    void persist_rest();
};

void sumcheck_prove_dev(zk_ctx* ctx, zk_transcript* tr, const ScStatement& S, Scratch& s);
uint64_t sumcheck_proof_len(uint32_t m, uint32_t K);

}  // namespace zk
