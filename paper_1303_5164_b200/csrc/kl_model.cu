// kl_model.cu -- batched Markov warp-state model + fused greedy selection (product path).
//
// One CTA per candidate (kind1, b1, kind2, b2).  Per candidate it builds the two solo chains and
// the joint chain of PAPER.md §4.4 in shared memory (fp64), solves each steady state with GTH
// (Grassmann-Taksar-Heyman state reduction: subtraction-free, so no pivoting is needed), and
// reduces Eq.4-8 and Eq.1.  The CTA that finishes last runs FindCoSchedule's selection (a9):
// per pair argmin dT over its maximal splits, then argmax CP over pairs.
//
// Readings: R1 P_ir = min(1, max(#ready,1)/L); R2 L(n) = L0 + a0 n/B + b0 with n
// the outstanding requests of the idle warps; R3 independent warps (binomial convolution);
// R4/R5 shared round and latency in the joint chain; R14 w = b * wpb / n_sched; R22 guard L > W.
#include <cuda_runtime.h>
#include <cstdint>
#include "kl_internal.h"

namespace {

constexpr int kMaxW = 16;                 // virtual-SM warps (64 warps / 4 schedulers)
constexpr int kMaxS = (kMaxW / 2 + 1) * (kMaxW / 2 + 1);   // 81 joint states at W_v = 16
constexpr int kThreads = 128;

// Binomial coefficients C(n,k), n <= 16 (exact in double).
__constant__ double c_binom[17][17];

__device__ __forceinline__ double binom_d(int n, int k) { return (k < 0 || k > n) ? 0.0 : c_binom[n][k]; }

__device__ double latency(const KlModelCfg& c, double n, int idle) {
    if (c.latency_mode == 1) return c.L0 + c.B / (c.a0 * (double)(idle > 1 ? idle : 1)) + c.b0;
    return c.L0 + c.a0 * n / c.B + c.b0;
}

// Round duration (R1) with the B200 pipe ceilings (R26): issue of all
// ready warps, each kernel's pipe time (ready / pi), pipes shared between kernels on the same
// pipe id; at least one cycle.
__device__ double round_dur(int r1, const KlModelKind* k1, int r2, const KlModelKind* k2) {
    double R = (double)(r1 + r2);
    const double p1 = k1 ? k1->pi : 1.0, p2 = k2 ? k2->pi : 1.0;
    if (k1 && k2 && k1->pipe != 0 && k1->pipe == k2->pipe) {
        R = fmax(R, r1 / p1 + r2 / p2);
    } else {
        R = fmax(R, r1 / p1);
        R = fmax(R, r2 / p2);
    }
    return fmax(R, 1.0);
}

// P_ir in a state of round duration R (R1); returns false if the guard L > W fails (R22).
__device__ bool p_ir(const KlModelCfg& c, double R, int idle, double n, double* out) {
    double L = latency(c, n, idle);
    if (!(L > (double)c.W)) return false;
    double p = R / L;
    *out = p < 1.0 ? p : 1.0;
    return true;
}

// One-kernel transition row from i idle of w (Eq.2 summed with binomial weights, R3).  The
// powers p^a (1-p)^(i-a) are built by repeated multiplication (no pow()), in the same (a, b)
// accumulation order as the oracle.
__device__ void row_of(int w, int i, double pir, double rm, double* row) {
    double pw[kMaxW + 1], qw[kMaxW + 1], rw[kMaxW + 1], sw[kMaxW + 1];
    pw[0] = qw[0] = rw[0] = sw[0] = 1.0;
    for (int t = 1; t <= w; ++t) {
        pw[t] = pw[t - 1] * pir;
        qw[t] = qw[t - 1] * (1.0 - pir);
        rw[t] = rw[t - 1] * rm;
        sw[t] = sw[t - 1] * (1.0 - rm);
    }
    for (int j = 0; j <= w; ++j) row[j] = 0.0;
    const int nr = w - i;
    for (int a = 0; a <= i; ++a) {
        const double pa = binom_d(i, a) * pw[a] * qw[i - a];
        for (int b = 0; b <= nr; ++b) row[i - a + b] += pa * (binom_d(nr, b) * rw[b] * sw[nr - b]);
    }
}

__device__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) s += red[i];
    return s;
}

// GTH steady state of the S x S row-stochastic matrix P (destroyed).  Returns false when a
// pivot sum is zero (reducible chain).
__device__ bool gth(double* P, int S, double* pi, double* red, int* flag) {
    for (int k = S - 1; k >= 1; --k) {
        double part = 0.0;
        for (int j = threadIdx.x; j < k; j += kThreads) part += P[k * S + j];
        double s = block_sum(part, red);
        if (!(s > 0.0)) return false;
        for (int i = threadIdx.x; i < k; i += kThreads) P[i * S + k] /= s;
        __syncthreads();
        for (int idx = threadIdx.x; idx < k * k; idx += kThreads) {
            int i = idx / k, j = idx - i * k;
            P[i * S + j] += P[i * S + k] * P[k * S + j];
        }
        __syncthreads();
    }
    // back substitution by warp 0: pi_j = sum_{i<j} pi_i P[i][j]
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0) pi[0] = 1.0;
        __syncwarp();
        for (int j = 1; j < S; ++j) {
            double part = 0.0;
            for (int i = threadIdx.x; i < j; i += 32) part += pi[i] * P[i * S + j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            if (threadIdx.x == 0) pi[j] = part;
            __syncwarp();
        }
    }
    __syncthreads();
    double part = 0.0;
    for (int i = threadIdx.x; i < S; i += kThreads) part += pi[i];
    double tot = block_sum(part, red);
    for (int i = threadIdx.x; i < S; i += kThreads) pi[i] /= tot;
    __syncthreads();
    (void)flag;
    return true;
}

// Solo IPC (Eq.4, denominator = elapsed cycles sum_i g_i R_i) of a kind at w warps on the
// virtual SM.
__device__ bool solo_ipc(const KlModelKind& k, int w, const KlModelCfg& c, double* P, double* pi,
                         double* red, double* out) {
    const int S = w + 1;
    __shared__ int s_ok;
    __shared__ double s_R[kMaxW + 1];
    if (threadIdx.x == 0) s_ok = 1;
    __syncthreads();
    for (int i = threadIdx.x; i < S; i += kThreads) {
        double pr;
        const double R = round_dur(w - i, &k, 0, nullptr);
        s_R[i] = R;
        if (!p_ir(c, R, i, (double)i * k.r, &pr)) { s_ok = 0; continue; }
        row_of(w, i, pr, k.rm, P + i * S);
    }
    __syncthreads();
    if (!s_ok) return false;
    if (!gth(P, S, pi, red, nullptr)) return false;
    double num = 0.0, den = 0.0;
    for (int i = threadIdx.x; i < S; i += kThreads) {
        if (i < w) num += pi[i] * (double)(w - i);
        den += pi[i] * s_R[i];
    }
    num = block_sum(num, red);
    den = block_sum(den, red);
    *out = num / den;
    __syncthreads();
    return true;
}

__device__ __forceinline__ double band(double x, double y) {
    double m = fmax(1.0, fmax(fabs(x), fabs(y)));
    return 1e-12 * m;
}

// a9 split order: argmin dT; ties (1e-12 band): larger C, more warps, smaller b1.
__device__ bool better_split(const kl_prediction& a, const KlCand& ca, const kl_prediction& b, const KlCand& cb,
                             int rule) {
    if (rule == 1) {   // ablation: highest predicted CP first
        double t = band(a.cp, b.cp);
        if (a.cp > b.cp + t) return true;
        if (a.cp < b.cp - t) return false;
    }
    double t = band(a.dT, b.dT);
    if (a.dT < b.dT - t) return true;
    if (a.dT > b.dT + t) return false;
    t = band(a.c, b.c);
    if (a.c > b.c + t) return true;
    if (a.c < b.c - t) return false;
    if (ca.warps != cb.warps) return ca.warps > cb.warps;
    return ca.b1 < cb.b1;
}

__global__ void __launch_bounds__(kThreads)
k_model_batch(const KlModelKind* __restrict__ kinds, const KlModelCfg cfg, const KlCand* __restrict__ cands,
              kl_prediction* preds, int n_pairs, const int32_t* __restrict__ pair_off,
              uint32_t* done_counter, KlDecision* dec) {
    extern __shared__ __align__(16) double smem_d[];
    double* P = smem_d;                    // kMaxS * kMaxS
    double* pi = P + kMaxS * kMaxS;        // kMaxS
    double* R = pi + kMaxS;                // kMaxS
    double* red = R + kMaxS;               // 8
    __shared__ int s_ok, s_last;
    __shared__ int s_best_pair[128];

    const KlCand cd = cands[blockIdx.x];
    const KlModelKind k1 = kinds[cd.k1], k2 = kinds[cd.k2];
    kl_prediction out = {};
    int status = 0;
    const int t1 = (int)cd.b1 * k1.wpb, t2 = (int)cd.b2 * k2.wpb;
    const int ts1 = k1.bsolo * k1.wpb, ts2 = k2.bsolo * k2.wpb;
    if (t1 % cfg.n_sched || t2 % cfg.n_sched || ts1 % cfg.n_sched || ts2 % cfg.n_sched) status = KL_EINFEASIBLE;
    const int w1 = t1 / cfg.n_sched, w2 = t2 / cfg.n_sched;
    const int ws1 = ts1 / cfg.n_sched, ws2 = ts2 / cfg.n_sched;
    const bool solo_query = (cd.b2 == 0);   // prediction of k1 alone at b1 (calibration)
    if (w1 < 1 || (w2 < 1 && !solo_query) || w1 + w2 > cfg.W || ws1 < 1 || ws1 > cfg.W || ws2 < 1 ||
        ws2 > cfg.W || (w1 + 1) * (w2 + 1) > kMaxS || cfg.W > kMaxW)
        status = KL_EINFEASIBLE;
    if (status == 0) {
        if (!solo_ipc(k1, ws1, cfg, P, pi, red, &out.solo1) || !solo_ipc(k2, ws2, cfg, P, pi, red, &out.solo2))
            status = KL_ENUMERIC;
    }
    if (status == 0) {
        const int S = (w1 + 1) * (w2 + 1);
        if (threadIdx.x == 0) s_ok = 1;
        __syncthreads();
        // joint chain: row (p,q) = outer product of the two one-kernel rows, both
        // evaluated with the shared round duration and latency of state (p,q)
        for (int s = threadIdx.x; s < S; s += kThreads) {
            const int p = s / (w2 + 1), q = s - p * (w2 + 1);
            double pr, r1[kMaxW + 1], r2[kMaxW + 1];
            R[s] = round_dur(w1 - p, &k1, w2 - q, solo_query ? nullptr : &k2);
            if (!p_ir(cfg, R[s], p + q, (double)p * k1.r + (double)q * k2.r, &pr)) { s_ok = 0; continue; }
            row_of(w1, p, pr, k1.rm, r1);
            row_of(w2, q, pr, k2.rm, r2);
            for (int pp = 0; pp <= w1; ++pp)
                for (int qq = 0; qq <= w2; ++qq) P[s * S + pp * (w2 + 1) + qq] = r1[pp] * r2[qq];
        }
        __syncthreads();
        if (!s_ok || !gth(P, S, pi, red, nullptr)) {
            status = KL_ENUMERIC;
        } else {
            // Eq.5-7 with R_(i,j) = joint round duration (R4)
            double den = 0.0, n1 = 0.0, n2 = 0.0;
            for (int s = threadIdx.x; s < S; s += kThreads) {
                const int p = s / (w2 + 1), q = s - p * (w2 + 1);
                den += pi[s] * R[s];
                if (p < w1) n1 += pi[s] * (double)(w1 - p);
                if (q < w2) n2 += pi[s] * (double)(w2 - q);
            }
            den = block_sum(den, red);
            n1 = block_sum(n1, red);
            n2 = block_sum(n2, red);
            out.ipc1 = n1 / den;
            out.ipc2 = n2 / den;
            out.c = out.ipc1 + out.ipc2;
            if (!solo_query) {
                out.cp = 1.0 - 1.0 / (out.ipc1 / out.solo1 + out.ipc2 / out.solo2);   // Eq.1
                out.dT = fabs(k1.ipb * (double)cd.b1 / out.ipc1 - k2.ipb * (double)cd.b2 / out.ipc2);  // Eq.8
            }
        }
    }
    out.status = status;
    if (threadIdx.x == 0) preds[blockIdx.x] = out;
    if (n_pairs <= 0) return;

    // ---- fused selection by the last CTA ---------------------------------------------------
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(done_counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int pr = threadIdx.x; pr < n_pairs; pr += kThreads) {
        int best = -1;
        kl_prediction bp;
        KlCand bc;
        for (int i = pair_off[pr]; i < pair_off[pr + 1]; ++i) {
            kl_prediction a = preds[i];
            if (a.status != 0) continue;
            KlCand ca = cands[i];
            if (best < 0 || better_split(a, ca, bp, bc, cfg.split_rule)) { best = i; bp = a; bc = ca; }
        }
        if (pr < 128) s_best_pair[pr] = best;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int best = -1;
        double bcp = 0.0;
        for (int pr = 0; pr < n_pairs && pr < 128; ++pr) {
            int i = s_best_pair[pr];
            if (i < 0) continue;
            double cp = preds[i].cp;
            if (best < 0 || cp > bcp + band(cp, bcp)) { best = i; bcp = cp; }
        }
        // (R25 "no profitable pair -> solo" is applied by the host with the configured cp_min)
        dec->cand = best;
        dec->cp = best >= 0 ? bcp : 0.0;
        dec->n_pairs = n_pairs;
        *done_counter = 0u;
        __threadfence_system();
        dec->done = 1;
    }
}

}  // namespace

int kl_dev_model_batch(const KlModelKind* kinds, KlModelCfg cfg, const KlCand* cands,
                       kl_prediction* preds, int n_pairs, const int32_t* pair_off,
                       uint32_t* done_counter, KlDecision* dec, void* stream) {
    if (cfg.n_cand <= 0) return 0;
    const size_t smem = sizeof(double) * (kMaxS * kMaxS + 3 * kMaxS + 8);
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_model_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        double tab[17][17] = {};
        for (int n = 0; n <= 16; ++n) {
            tab[n][0] = 1.0;
            for (int k = 1; k <= n; ++k) tab[n][k] = tab[n - 1][k - 1] + (k <= n - 1 ? tab[n - 1][k] : 0.0);
        }
        e = cudaMemcpyToSymbol(c_binom, tab, sizeof(tab));
        if (e != cudaSuccess) return (int)e;
        attr = true;
    }
    k_model_batch<<<cfg.n_cand, kThreads, smem, (cudaStream_t)stream>>>(kinds, cfg, cands, preds, n_pairs,
                                                                      pair_off, done_counter, dec);
    return (int)cudaGetLastError();
}
