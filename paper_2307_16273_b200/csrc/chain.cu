// chain.cu — SURVEY §8(f) N3: the claim merge of DESIGN.md D25 (Eq. sc-reindex, in its
// general form; Protocol 1 line 8), the step that chains a FAC4DNN window: every claim the
// operation families leave on views of one tensor family (the matmul claims Y~(w, u1, u3) and the
// operand finals) is reduced to ONE claim on the tensor family's stack.
//
// X: N = 2^n slices of rows x cols int32 (a point is (col bits, row bits, slice bits), D2), possibly
// virtual (A and G_Z are formed from the zkReLU words on the fly, Lemma 1, P:L546-547 — the tensors
// "anchored by the commitment of aux").  Claim k: c_k = X_k~(v_k, u_k) on a view (slot j holds
// slice map_k[j]).  With rho_k drawn by the verifier:
//   phase A: sum_k rho_k c_k = sum_{i,k} P(i,k) Rt(i,k), P = rho_k S_k(i), Rt = X_i~(v_k), over n + kappa
//            variables (i first);  Rt is formed by row dots against beta(v_k.cols) (lazy int32 x Fr) and
//            a dot over rows against beta(v_k.rows);
//   phase B: Rt~(r_i, r_k) = sum_y Wy(y) Xr(y), Wy = sum_k beta(r_k, k) beta(v_k, y), Xr = sum_i
//            beta(r_i, i) X(i, y) (one column-sum pass over the stack), over the d inner variables.
// Both phases run on the product-sumcheck engine (rows a4-a6).  Everything is stream-ordered on the
// context stream: no host synchronisation, no pageable copies (maps travel as kernel parameters).
#include <cstring>
#include <type_traits>
#include <vector>

#include "sumcheck.cuh"
#include "tables.cuh"

using namespace zk;

namespace zk {

// defined in n1.cu / tables.cu
__global__ void k_canon_to_mont(const uint8_t* in, uint32_t n, fr_t* out);
__global__ void k_lincomb(const fr_t* a, const fr_t* b, uint32_t K, fr_t* out);
__global__ void k_rowdot_fr(const fr_t* T, uint64_t nrows, uint32_t cols, const fr_t* w, fr_t* out);

constexpr uint32_t CM_MAX_K = 8, CM_MAX_SLOTS = 2048;
struct CmMaps {
    uint32_t K, N;
    uint32_t off[CM_MAX_K + 1];      // slot ranges of the views in idx
    uint32_t idx[CM_MAX_SLOTS];      // slot -> slice (0xffffffff: empty)
};

// P[k * N + map_k[j]] = rho_k * E_k[j]  (maps injective per view, so every (k, j) owns its target)
__global__ void k_cm_scatter(CmMaps M, const fr_t* E, const fr_t* rho, fr_t* P) {
    const uint32_t total = M.off[M.K];
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        uint32_t k = 0;
        while (t >= M.off[k + 1]) k++;
        const uint32_t i = M.idx[t];
        if (i == 0xffffffffu) continue;
        fr_store(&P[(uint64_t)k * M.N + i], fr_mul(fr_load(&rho[k]), fr_load(&E[t])));
    }
}


// Xr[y] = sum_i beta(r_i, i) X(i, y): the column sums of the [N][D] stack (E2 = beta(r_i) scaled by R)
template <class Load>
static void cm_colsum(zk_ctx* ctx, Load load, uint64_t N, uint64_t D, const fr_t* E2, fr_t* out, Scratch& s) {
    if constexpr (std::is_same_v<Load, LoadPlain>) {
        if (D <= 0xffffffffull && colsum_tc_ok(1, (uint32_t)N, (uint32_t)D)) {   // a stored stack: tensor cores (TMA)
            colsum_tc(ctx, load.p, 1, (uint32_t)N, (uint32_t)D, E2, out, s);
            return;
        }
    }
    const uint64_t blocks = (D + 127) / 128;
    const unsigned int grid = (unsigned int)(blocks < (uint64_t)ctx->num_sms * 7 ? blocks : (uint64_t)ctx->num_sms * 7);
    ZK_LAUNCH(ctx, k_colsum_i32<Load>, grid, 128, 0, load, (uint64_t)1, (uint32_t)N, (uint32_t)D, E2, out, 1u,
              (uint32_t*)nullptr);
}

static inline uint32_t n_log(uint64_t N) {
    uint32_t l = 0;
    while ((1ull << l) < N) l++;
    return l;
}

// Rt(i, k) for one claim: T[i * rows + row] = sum_col beta(v.cols)[col] X[i][row][col]; Rt = T . beta(v.rows)
// (Ec = beta(v.cols) scaled by R, Er = beta(v.rows): built by the caller's batched eq-table launches)
template <class Load>
static void cm_slice_mles(zk_ctx* ctx, Load load, uint64_t N, uint32_t lr, uint32_t lc, const fr_t* Ec, const fr_t* Er,
                          fr_t* out, Scratch& s) {
    const uint64_t rows = 1ull << lr, cols = 1ull << lc;
    fr_t* T = s.alloc<fr_t>(N * rows);
    if constexpr (std::is_same_v<Load, LoadPlain>) {
        if (rowdot_tc_ok(N * rows, (uint32_t)cols)) {   // a stored stack: the row dots on the tensor cores (TMA)
            rowdot_tc(ctx, load.p, N * rows, (uint32_t)cols, Ec, T, N * rows, n_log(N) + lr, 1, s);
            ZK_LAUNCH(ctx, k_rowdot_fr, grid_for(ctx, N * 32, 256, 8), 256, 0, (const fr_t*)T, N, (uint32_t)rows, Er, out);
            return;
        }
    }
    ZK_LAUNCH(ctx, k_rowdot_i32<Load>, grid_for(ctx, N * rows * 32, 256, 8), 256, 0, load, N * rows, (uint32_t)cols,
              Ec, T, N * rows, (uint32_t)(n_log(N) + lr), (uint64_t)1);
    // the row dots are in natural order (inner = nrows: identity map)
    ZK_LAUNCH(ctx, k_rowdot_fr, grid_for(ctx, N * 32, 256, 8), 256, 0, (const fr_t*)T, N, (uint32_t)rows, Er, out);
}

// W[y] = sum_k T_k[y] over K tables of D entries (phase B's sum of the scaled eq tables)
struct CmTabs {
    const fr_t* t[64];
};
__global__ void k_cm_sum_tables(CmTabs T, uint32_t K, uint64_t D, fr_t* W) {
    for (uint64_t y = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; y < D; y += (uint64_t)gridDim.x * blockDim.x) {
        fr_t acc = fr_load(&T.t[0][y]);
        for (uint32_t k = 1; k < K; k++) acc = fr_add(acc, fr_load(&T.t[k][y]));
        fr_store(&W[y], acc);
    }
}

struct CmLayout {
    uint64_t la, lb, off_b, off_pa, off_pb, off_pt, off_c, total;
};
static CmLayout cm_layout(uint32_t n, uint32_t kap, uint32_t d) {
    CmLayout L;
    L.la = sumcheck_proof_len(n + kap, 2);
    L.lb = sumcheck_proof_len(d, 2);
    L.off_b = L.la;
    L.off_pa = (L.la + L.lb + 15) & ~15ull;
    L.off_pb = L.off_pa + 32ull * (n + kap);
    L.off_pt = L.off_pb + 32ull * d;
    L.off_c = L.off_pt + 32ull * (d + n);
    L.total = L.off_c + 32;
    return L;
}

template <class Load>
static void claim_merge_dev(zk_ctx* ctx, zk_transcript* tr, Load load, uint32_t n, uint32_t lr, uint32_t lc,
                            const CmMaps& M, const uint32_t* nk, const uint8_t* d_pts, const uint8_t* d_claims,
                            uint8_t* d_out, Scratch& s) {
    const uint32_t K = M.K, d = lr + lc;
    uint32_t kap = 0;
    while ((1u << kap) < K) kap++;
    const uint64_t N = 1ull << n, D = 1ull << d, NA = N << kap;
    const CmLayout L = cm_layout(n, kap, d);
    // header, claims, rho (transcript D25)
    std::vector<uint8_t> hb(4 * (3 + K));
    const uint32_t h3[3] = {n, d, K};
    for (uint32_t i = 0; i < 3 + K; i++) {
        const uint32_t v = i < 3 ? h3[i] : nk[i - 3];
        for (int b = 0; b < 4; b++) hb[4 * i + b] = (uint8_t)(v >> (8 * b));
    }
    tr_absorb_host(tr, "cm/hdr", hb.data(), hb.size());
    fr_t* cl = s.alloc<fr_t>(K);
    ZK_LAUNCH(ctx, k_canon_to_mont, 1, 32, 0, d_claims, K, cl);
    ZK_LAUNCH(ctx, k_tr_absorb_frs, 1, 32, 0, tr->d_st, make_tag("cm/claims"), (const fr_t*)cl, K, (uint8_t*)nullptr);
    fr_t* rho = s.alloc<fr_t>(K);
    tr_challenges_dev(tr, "cm/rho", K, rho, nullptr);
    // the points (per claim: v_k, d elements, then u_k, nk elements), Montgomery
    uint32_t npts = 0;
    std::vector<uint32_t> poff(K);
    for (uint32_t k = 0; k < K; k++) {
        poff[k] = npts;
        npts += d + nk[k];
    }
    fr_t* pts = s.alloc<fr_t>(npts);
    ZK_LAUNCH(ctx, k_canon_to_mont, grid_for(ctx, npts, 128, 1), 128, 0, d_pts, npts, pts);
    // phase A tables (flat k * N + i)
    fr_t* P = s.alloc_zero<fr_t>(NA);
    fr_t* Rt = s.alloc_zero<fr_t>(NA);
    fr_t* E = s.alloc<fr_t>(M.off[K] ? M.off[K] : 1);
    // every eq table of phase A in batched launches: per claim the slot table, and the column (R-scaled) and
    // row tables of its inner point
    std::vector<EqJob> jobs;
    std::vector<fr_t*> Ec(K), Er(K);
    for (uint32_t k = 0; k < K; k++) {
        Ec[k] = s.alloc<fr_t>(1ull << lc);
        Er[k] = s.alloc<fr_t>(1ull << lr);
        jobs.push_back(EqJob{pts + poff[k] + d, nk[k], nullptr, 0, E + M.off[k]});
        jobs.push_back(EqJob{pts + poff[k], lc, nullptr, 1, Ec[k]});
        jobs.push_back(EqJob{pts + poff[k] + lc, lr, nullptr, 0, Er[k]});
    }
    eq_tables_batch(ctx, (uint32_t)jobs.size(), jobs.data(), s);
    for (uint32_t k = 0; k < K; k++) cm_slice_mles(ctx, load, N, lr, lc, Ec[k], Er[k], Rt + (uint64_t)k * N, s);
    ZK_LAUNCH(ctx, k_cm_scatter, grid_for(ctx, M.off[K], 128, 1), 128, 0, M, (const fr_t*)E, (const fr_t*)rho, P);
    ScStatement A;
    memset(&A, 0, sizeof A);
    A.m = n + kap;
    A.K = 2;
    A.tables[0] = P;
    A.tables[1] = Rt;
    A.d_claim = s.alloc<fr_t>(1);
    A.claim_given = true;
    ZK_LAUNCH(ctx, k_lincomb, 1, 1, 0, (const fr_t*)rho, (const fr_t*)cl, K, A.d_claim);
    A.d_proof = d_out;
    A.d_r = s.alloc<fr_t>(n + kap);
    A.d_point = d_out + L.off_pa;
    A.d_finals = s.alloc<fr_t>(2);
    sumcheck_prove_dev(ctx, tr, A, s);
    // phase B: Xr = sum_i beta(r_i, i) X(i, .), Wy = sum_k beta(r_k, k) beta(v_k, .)
    fr_t* Ei = s.alloc<fr_t>(N);
    eq_table_r2_dev(ctx, A.d_r, n, Ei, s);
    fr_t* Xr = s.alloc<fr_t>(D);
    cm_colsum(ctx, load, N, D, Ei, Xr, s);
    fr_t* Bk = s.alloc<fr_t>(1ull << kap);
    eq_table_dev(ctx, A.d_r + n, kap, nullptr, Bk, s);
    fr_t* Wy = s.alloc<fr_t>(D);
    // Wy = sum_k beta(r_k, k) beta(v_k, .): the K tables scaled by beta(r_k, k) in batched launches, then summed
    ZK_REQUIRE(K <= 64, ZK_ERR_ARG, "claim merge: at most 64 claims");
    CmTabs tabs;
    std::vector<EqJob> bj;
    for (uint32_t k = 0; k < K; k++) {
        fr_t* Ev = s.alloc<fr_t>(D);
        tabs.t[k] = Ev;
        bj.push_back(EqJob{pts + poff[k], d, Bk + k, 0, Ev});
    }
    eq_tables_batch(ctx, K, bj.data(), s);
    ZK_LAUNCH(ctx, k_cm_sum_tables, grid_for(ctx, D, 256, 4), 256, 0, tabs, K, D, Wy);
    ScStatement B;
    memset(&B, 0, sizeof B);
    B.m = d;
    B.K = 2;
    B.tables[0] = Wy;
    B.tables[1] = Xr;
    B.d_claim = A.d_finals + 1;    // Rt~(r_i, r_k)
    B.claim_given = true;
    B.d_proof = d_out + L.off_b;
    B.d_r = s.alloc<fr_t>(d);
    B.d_point = d_out + L.off_pb;
    B.d_finals = s.alloc<fr_t>(2);
    sumcheck_prove_dev(ctx, tr, B, s);
    // the one claim left on the stack: X~(r_B, r_A[:n]) = Xr~(r_B)
    ZK_CUDA(cudaMemcpyAsync(d_out + L.off_pt, d_out + L.off_pb, 32ull * d, cudaMemcpyDeviceToDevice, ctx->stream));
    if (n)
        ZK_CUDA(cudaMemcpyAsync(d_out + L.off_pt + 32ull * d, d_out + L.off_pa, 32ull * n, cudaMemcpyDeviceToDevice,
                                ctx->stream));
    to_canonical_dev(ctx, B.d_finals + 1, 1, d_out + L.off_c);
}

}  // namespace zk

extern "C" {

zk_status zk_claim_merge_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_X, const int32_t* d_X2, uint32_t source,
                             uint32_t R, uint32_t n, uint32_t log_rows, uint32_t log_cols, uint32_t K,
                             const zk_cm_view* views, const uint8_t* d_pts, const uint8_t* d_claims, uint8_t* d_out,
                             uint64_t* out_len) {
    if (!ctx) return ZK_ERR_ARG;
    try {
        ZK_CUDA(cudaSetDevice(ctx->device));
        ZK_REQUIRE(K >= 1 && K <= CM_MAX_K && n <= 16 && log_rows + log_cols >= 1 && log_rows + log_cols <= 30 &&
                       log_cols <= 16 && log_rows <= 16,
                   ZK_ERR_ARG, "bad claim-merge shape");
        uint32_t kap = 0;
        while ((1u << kap) < K) kap++;
        ZK_REQUIRE(n + kap >= 1, ZK_ERR_ARG, "a single claim on a single slice needs no merge");
        const CmLayout L = cm_layout(n, kap, log_rows + log_cols);
        ZK_REQUIRE(d_out || out_len, ZK_ERR_ARG, "null output");
        if (!d_out) {
            *out_len = L.total;
            return ZK_OK;
        }
        ZK_REQUIRE(out_len && *out_len >= L.total, ZK_ERR_ARG, "d_out too small (*out_len < the required size)");
        *out_len = L.total;
        ZK_REQUIRE(((uintptr_t)d_out & 15) == 0, ZK_ERR_ARG, "d_out must be 16-byte aligned");
        ZK_REQUIRE(tr && d_X && views && d_pts && d_claims, ZK_ERR_ARG, "null argument");
        ZK_REQUIRE(source <= 3 && (source != 2 || d_X2) && (source == 0 || (R >= 1 && R <= 32)) &&
                       (source != 3 || n == 0),
                   ZK_ERR_ARG, "bad source");
        CmMaps M;
        memset(&M, 0, sizeof M);
        M.K = K;
        M.N = 1u << n;
        std::vector<uint32_t> nk(K);
        std::vector<uint8_t> seen(1ull << n);
        for (uint32_t k = 0; k < K; k++) {
            nk[k] = views[k].logN;
            ZK_REQUIRE(views[k].logN <= 16 && views[k].map, ZK_ERR_ARG, "bad view");
            const uint32_t ns = 1u << views[k].logN;
            ZK_REQUIRE(M.off[k] + ns <= CM_MAX_SLOTS, ZK_ERR_ARG, "too many view slots");
            M.off[k + 1] = M.off[k] + ns;
            std::fill(seen.begin(), seen.end(), 0);
            for (uint32_t j = 0; j < ns; j++) {
                const uint32_t i = views[k].map[j];
                M.idx[M.off[k] + j] = i;
                if (i == 0xffffffffu) continue;
                ZK_REQUIRE(i < M.N, ZK_ERR_RANGE, "view slot outside the stack");
                ZK_REQUIRE(!seen[i], ZK_ERR_ARG, "view map not injective");
                seen[i] = 1;
            }
        }
        Scratch s(ctx);
        if (source == 0)
            claim_merge_dev(ctx, tr, LoadPlain{d_X}, n, log_rows, log_cols, M, nk.data(), d_pts, d_claims, d_out, s);
        else if (source == 1)
            claim_merge_dev(ctx, tr, LoadReluA{d_X, R}, n, log_rows, log_cols, M, nk.data(), d_pts, d_claims, d_out, s);
        else if (source == 2)
            claim_merge_dev(ctx, tr, LoadReluGZ{d_X, d_X2, R}, n, log_rows, log_cols, M, nk.data(), d_pts, d_claims,
                            d_out, s);
        else   // the rescale's aux bits (D26): one slice of 2^log_rows entries x 2^log_cols bit columns
            claim_merge_dev(ctx, tr, LoadBits{d_X, log_cols, R}, n, log_rows, log_cols, M, nk.data(), d_pts,
                            d_claims, d_out, s);
    } catch (const ::zk::ZkError& e) {
        ctx->err = e.msg;
        return e.st;
    } catch (const std::exception& e) {
        ctx->err = e.what();
        return ZK_ERR_INTERNAL;
    }
    return ZK_OK;
}

}  // extern "C"
