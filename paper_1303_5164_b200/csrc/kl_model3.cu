// kl_model3.cu -- the general batched model (product path): f1 three-state (coalesced /
// uncoalesced) chains and/or thread blocks as the modelling unit
// (P:1042-1051), for every candidate of a batch; same predictions and fused selection (a9) as
// the two-state kernel of kl_model.cu, which stays the fast path when neither is configured.
//
// Per kind (readings R27 and R13 in DESIGN.md §3): Rm, r (requests per coalesced memory
// instruction), uc (uncoalesced fraction of memory instructions), ru (requests per uncoalesced
// one), units of g warps.  A kind with `three` set has states (c, u) = coalesced-idle and
// uncoalesced-idle units, c + u <= m; otherwise (c) only.  One kernel's row from (c, u) with
// ready = m - c - u units:
//   T((c,u) -> (c',u')) = sum_{x,y} M(x,y) A(c'-x) Bu(u'-y),
//   A(j) = Binomial(c, P_c) mass at c - j returns, Bu(j) likewise with P_u,
//   M(x,y) = multinomial(ready; x coalesced stalls, y uncoalesced stalls) with probabilities
//            Rm(1-uc), Rm uc, 1-Rm.
// The round sees g x ready warps (R1, R26), n = sum g (c r + u ru) outstanding requests,
// L_c = L0 + a0 n/B + b0 (R2), L_u = L_c + a0 (ru - r)/B, P_x = min(1, R/L_x), guard L_c > W
// (R22); IPC counts g instructions per ready unit (Eq.4-7).
//
// Layout: one CTA (8 warps) per candidate.  Its chains live in global scratch (P row-major
// S x S, then pi, R, 1/s_k), so the state count is bounded by memory, not shared memory (S up
// to 2025 at 8+8 warps in warp granularity; 225 in block granularity).  Rows are built one warp
// per source state with per-warp shared tables; the steady state is GTH on a 16 x 16 thread
// tile with one barrier per eliminated state, as in kl_model.cu.
#include <cuda_runtime.h>
#include <cstdint>
#include "kl_internal.h"
#include "kl_model_common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kNW = kThreads / 32;
constexpr int kMaxU = 16;                         // units per kind on the virtual SM
constexpr int kMaxN = (kMaxU + 1) * (kMaxU + 2) / 2;   // 153 states of one kind

__constant__ double c_binom3[kMaxU + 1][kMaxU + 1];

struct Kin {                  // one kernel of a chain
    const KlModelKind* k;     // null: absent (solo chain)
    int m, g, three, n;       // units, warps per unit, three-state, number of states
};

__device__ __forceinline__ int nstates(int m, int three) { return three ? (m + 1) * (m + 2) / 2 : m + 1; }

// (c, u) of state t of a kind (index order c-major, as the oracle's idx3)
__device__ __forceinline__ void decode(const Kin& K, int t, int* c, int* u) {
    if (!K.three) { *c = t; *u = 0; return; }
    int cc = 0, base = 0;
    while (base + (K.m - cc + 1) <= t) { base += K.m - cc + 1; ++cc; }
    *c = cc;
    *u = t - base;
}

__device__ __forceinline__ double pw(double x, int e) {
    double r = 1.0;
    for (int i = 0; i < e; ++i) r *= x;
    return r;
}

struct WarpTab {              // per-warp shared scratch for one kernel's row
    double A[kMaxU + 1], Bu[kMaxU + 1];
    double M[(kMaxU + 1) * (kMaxU + 1)];
};

// Row of kernel K from (c, u) into out[0..K.n) (shared), one warp.
__device__ void kind_row(const Kin& K, int c, int u, double pc, double pu, WarpTab* T, double* out,
                         const double (*binom)[kMaxU + 1]) {
    const int lane = threadIdx.x & 31, ready = K.m - c - u, rp = ready + 1;
    const double rm = K.k->rm, uc = K.three ? K.k->uc : 0.0;
    const double sc = rm * (1.0 - uc), su = rm * uc, st = 1.0 - rm;
    for (int j = lane; j <= c; j += 32) T->A[j] = binom[c][j] * pw(1.0 - pc, j) * pw(pc, c - j);
    for (int j = lane; j <= u; j += 32) T->Bu[j] = binom[u][j] * pw(1.0 - pu, j) * pw(pu, u - j);
    for (int e = lane; e < rp * rp; e += 32) {
        const int x = e / rp, y = e - x * rp;
        T->M[e] = (x + y <= ready && (K.three || y == 0))
                      ? binom[ready][x] * binom[ready - x][y] * pw(sc, x) * pw(su, y) * pw(st, ready - x - y)
                      : 0.0;
    }
    __syncwarp();
    for (int t = lane; t < K.n; t += 32) {
        int c2, u2;
        decode(K, t, &c2, &u2);
        double s = 0.0;
        const int x0 = c2 - c > 0 ? c2 - c : 0, x1 = c2 < ready ? c2 : ready;
        for (int x = x0; x <= x1; ++x) {
            const int y0 = u2 - u > 0 ? u2 - u : 0;
            const int y1 = u2 < ready - x ? u2 : ready - x;
            const double ax = T->A[c2 - x];
            for (int y = y0; y <= y1; ++y) s += T->M[x * rp + y] * ax * T->Bu[u2 - y];
        }
        out[t] = s;
    }
    __syncwarp();
}

__device__ __forceinline__ double warp_sum3(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ double block_sum3(double v, double* red) {
    v = warp_sum3(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < kNW; ++i) s += red[i];
    return s;
}

struct ChainIpc { double a, b; };

// Chain of kernels K1 (and K2 if present) in global scratch; IPCs by Eq.4-7.
__device__ int chain_general(const Kin& K1, const Kin& K2, const KlModelCfg& cfg, double* P, double* pi,
                             double* Rs, double* inv_s, double* red, WarpTab* tabs, double (*rows)[2][kMaxN],
                             const double (*binom)[kMaxU + 1], ChainIpc* out) {
    const int n1 = K1.n, n2 = K2.k ? K2.n : 1, S = n1 * n2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ int s_bad;
    __shared__ double s_piv[2], s_inv[2];
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    // ---- chain build: one warp per source state
    for (int s = warp; s < S; s += kNW) {
        const int s1 = s / n2, s2 = s - s1 * n2;
        int c1, u1, c2 = 0, u2 = 0;
        decode(K1, s1, &c1, &u1);
        if (K2.k) decode(K2, s2, &c2, &u2);
        const int rd1 = K1.m - c1 - u1, rd2 = K2.k ? K2.m - c2 - u2 : 0;
        const double R = round_dur(K1.g * rd1, K1.k, K2.g * rd2, K2.k);
        const int idle = K1.g * (c1 + u1) + (K2.k ? K2.g * (c2 + u2) : 0);
        const double n = K1.g * (c1 * K1.k->r + u1 * K1.k->ru) + (K2.k ? K2.g * (c2 * K2.k->r + u2 * K2.k->ru) : 0.0);
        const double Lc = latency(cfg, n, idle);
        if (!(Lc > (double)cfg.W)) {
            if (lane == 0) s_bad = 1;
            continue;
        }
        if (lane == 0) Rs[s] = R;
        const double Lu1 = Lc + cfg.a0 * (K1.k->ru - K1.k->r) / cfg.B;
        kind_row(K1, c1, u1, fmin(1.0, R / Lc), fmin(1.0, R / Lu1), &tabs[warp], rows[warp][0], binom);
        if (K2.k) {
            const double Lu2 = Lc + cfg.a0 * (K2.k->ru - K2.k->r) / cfg.B;
            kind_row(K2, c2, u2, fmin(1.0, R / Lc), fmin(1.0, R / Lu2), &tabs[warp], rows[warp][1], binom);
        } else if (lane == 0) {
            rows[warp][1][0] = 1.0;
        }
        __syncwarp();
        double* row = P + (size_t)s * S;
        for (int t1 = 0; t1 < n1; ++t1) {
            const double v1 = rows[warp][0][t1];
            for (int t2 = lane; t2 < n2; t2 += 32) row[t1 * n2 + t2] = v1 * rows[warp][1][t2];
        }
        __syncwarp();
    }
    __syncthreads();
    if (s_bad) return KL_ENUMERIC;
    // ---- GTH (see kl_model.cu): column k unscaled, 1/s_k applied in the back substitution
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    if (warp == 0) {
        double part = 0.0;
        for (int j = lane; j < S - 1; j += 32) part += P[(size_t)(S - 1) * S + j];
        part = warp_sum3(part);
        if (lane == 0) {
            s_piv[(S - 1) & 1] = part;
            s_inv[(S - 1) & 1] = 1.0 / part;
        }
    }
    __syncthreads();
    for (int k = S - 1; k >= 1; --k) {
        const double sk = s_piv[k & 1];
        if (!(sk > 0.0)) return KL_ENUMERIC;
        const double inv = s_inv[k & 1];
        if (threadIdx.x == 0) inv_s[k] = inv;
        const double* rk = P + (size_t)k * S;
        for (int i = ty; i < k; i += 16) {
            double* ri = P + (size_t)i * S;
            const double a = ri[k] * inv;
            for (int j = tx; j < k; j += 16) ri[j] = fma(a, rk[j], ri[j]);
        }
        if (warp == (((k - 1) & 15) >> 1)) {
            double part = 0.0;
            if (ty == ((k - 1) & 15)) {
                const double* rp = P + (size_t)(k - 1) * S;
                for (int j = tx; j < k - 1; j += 16) part += rp[j];
            }
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            if (tx == 0 && ty == ((k - 1) & 15)) {
                s_piv[(k - 1) & 1] = part;
                s_inv[(k - 1) & 1] = 1.0 / part;
            }
        }
        __syncthreads();
    }
    // back substitution by warp 0, pi[] as the column accumulators
    if (warp == 0) {
        for (int m = lane; m < S; m += 32) pi[m] = 0.0;
        __syncwarp();
        double tot = 0.0;
        for (int j = 0; j < S; ++j) {
            const double pj = j == 0 ? 1.0 : pi[j] * inv_s[j];
            tot += pj;
            __syncwarp();
            if (lane == 0) pi[j] = pj;
            const double* rj = P + (size_t)j * S;
            for (int m = j + 1 + lane; m < S; m += 32) pi[m] = fma(pj, rj[m], pi[m]);
            __syncwarp();
        }
        if (lane == 0) red[kNW] = tot;
    }
    __syncthreads();
    const double tot = red[kNW];
    double den = 0.0, na = 0.0, nb = 0.0;
    for (int s = threadIdx.x; s < S; s += kThreads) {
        const int s1 = s / n2, s2 = s - s1 * n2;
        int c1, u1, c2 = 0, u2 = 0;
        decode(K1, s1, &c1, &u1);
        if (K2.k) decode(K2, s2, &c2, &u2);
        const double g = pi[s] / tot;
        den += g * Rs[s];
        na += g * (double)(K1.g * (K1.m - c1 - u1));
        if (K2.k) nb += g * (double)(K2.g * (K2.m - c2 - u2));
    }
    den = block_sum3(den, red);
    na = block_sum3(na, red);
    nb = block_sum3(nb, red);
    out->a = na / den;
    out->b = nb / den;
    __syncthreads();
    return KL_OK;
}

// Kernel descriptor of kind k at w warps on the virtual SM (0 if not representable).
__device__ bool make_kin(const KlModelKind* k, int w, Kin* K) {
    K->k = k;
    K->g = k->g > 0 ? k->g : 1;
    if (w % K->g) return false;
    K->m = w / K->g;
    K->three = k->three;
    if (K->m < 1 || K->m > kMaxU) return false;
    K->n = nstates(K->m, K->three);
    return true;
}

__global__ void __launch_bounds__(kThreads)
k_model_general(const KlModelKind* __restrict__ kinds, const KlModelCfg cfg, const KlCand* __restrict__ cands,
                kl_prediction* preds, int n_pairs, const int32_t* __restrict__ pair_off, uint32_t* done_counter,
                KlDecision* dec, double* scratch, const int64_t* __restrict__ scratch_off) {
    __shared__ double s_binom[kMaxU + 1][kMaxU + 1];
    __shared__ WarpTab tabs[kNW];
    __shared__ double rows[kNW][2][kMaxN];
    __shared__ double red[kNW + 1];
    for (int x = threadIdx.x; x < (kMaxU + 1) * (kMaxU + 1); x += kThreads)
        s_binom[x / (kMaxU + 1)][x % (kMaxU + 1)] = c_binom3[x / (kMaxU + 1)][x % (kMaxU + 1)];
    __syncthreads();

    const KlCand cd = cands[blockIdx.x];
    const KlModelKind* k1 = kinds + cd.k1;
    const KlModelKind* k2 = kinds + cd.k2;
    kl_prediction out = {};
    int status = 0;
    const int t1 = (int)cd.b1 * k1->wpb, t2 = (int)cd.b2 * k2->wpb;
    const int ts1 = k1->bsolo * k1->wpb, ts2 = k2->bsolo * k2->wpb;
    if (t1 % cfg.n_sched || t2 % cfg.n_sched || ts1 % cfg.n_sched || ts2 % cfg.n_sched) status = KL_EINFEASIBLE;
    const int w1 = t1 / cfg.n_sched, w2 = t2 / cfg.n_sched;
    const int ws1 = ts1 / cfg.n_sched, ws2 = ts2 / cfg.n_sched;
    const bool solo_query = (cd.b2 == 0);
    Kin J1, J2, S1, S2, none{};
    none.k = nullptr;
    if (w1 < 1 || (w2 < 1 && !solo_query) || w1 + w2 > cfg.W || ws1 < 1 || ws1 > cfg.W || ws2 < 1 ||
        ws2 > cfg.W || cfg.W > kMaxU * 4)
        status = KL_EINFEASIBLE;
    if (status == 0 && (!make_kin(k1, w1, &J1) || (!solo_query && !make_kin(k2, w2, &J2)) ||
                        !make_kin(k1, ws1, &S1) || !make_kin(k2, ws2, &S2)))
        status = KL_EINFEASIBLE;
    double* base = scratch + scratch_off[blockIdx.x];
    ChainIpc co{};
    for (int pass = 0; pass < 3 && status == 0; ++pass) {
        const Kin& A = pass == 0 ? S1 : (pass == 1 ? S2 : J1);
        const Kin& B = pass < 2 ? none : (solo_query ? none : J2);
        const int S = A.n * (B.k ? B.n : 1);
        double* P = base;
        double* pi = P + (size_t)S * S;
        double* Rs = pi + S;
        double* inv_s = Rs + S;
        status = chain_general(A, B, cfg, P, pi, Rs, inv_s, red, tabs, rows, s_binom, &co);
        if (status) break;
        if (pass == 0) out.solo1 = co.a;
        if (pass == 1) out.solo2 = co.a;
        if (pass == 2) {
            out.ipc1 = co.a;
            out.ipc2 = co.b;
            out.c = co.a + co.b;
            if (!solo_query) {
                out.cp = 1.0 - 1.0 / (out.ipc1 / out.solo1 + out.ipc2 / out.solo2);   // Eq.1
                out.dT = fabs(k1->ipb * (double)cd.b1 / out.ipc1 - k2->ipb * (double)cd.b2 / out.ipc2);  // Eq.8
            }
        }
    }
    out.status = status;
    if (threadIdx.x == 0) {
        preds[blockIdx.x] = out;
        if (cfg.preds_host) cfg.preds_host[blockIdx.x] = out;   // the host reads these (mapped)
        if (cfg.cands_dev) cfg.cands_dev[blockIdx.x] = cd;
    }
    if (n_pairs <= 0) return;
    select_last<kThreads>(cfg, kinds, cfg.cands_dev ? cfg.cands_dev : cands, preds, n_pairs, pair_off, done_counter, dec);
}

}  // namespace

int kl_dev_model3_init() {
    double tab[kMaxU + 1][kMaxU + 1] = {};
    for (int n = 0; n <= kMaxU; ++n) {
        tab[n][0] = 1.0;
        for (int k = 1; k <= n; ++k) tab[n][k] = tab[n - 1][k - 1] + (k <= n - 1 ? tab[n - 1][k] : 0.0);
    }
    cudaError_t e = cudaMemcpyToSymbol(c_binom3, tab, sizeof(tab));
    if (e != cudaSuccess) return (int)e;
    cudaFuncAttributes fa;
    return (int)cudaFuncGetAttributes(&fa, k_model_general);
}

int kl_dev_model_general(const KlModelKind* kinds, KlModelCfg cfg, const KlCand* cands, kl_prediction* preds,
                         int n_pairs, const int32_t* pair_off, uint32_t* done_counter, KlDecision* dec,
                         double* scratch, const int64_t* scratch_off, void* stream) {
    if (cfg.n_cand <= 0) return 0;
    static bool init = false;
    if (!init) {
        int e = kl_dev_model3_init();
        if (e) return e;
        init = true;
    }
    k_model_general<<<cfg.n_cand, kThreads, 0, (cudaStream_t)stream>>>(kinds, cfg, cands, preds, n_pairs, pair_off,
                                                                       done_counter, dec, scratch, scratch_off);
    return (int)cudaGetLastError();
}
