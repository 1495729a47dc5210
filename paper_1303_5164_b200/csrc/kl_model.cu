// kl_model.cu -- batched Markov warp-state model + fused greedy selection (product path).
//
// One CTA (8 warps) per candidate (kind1, b1, kind2, b2).  Per candidate it builds the two solo
// chains and the joint chain of PAPER.md §4.4 in shared memory (fp64, one warp per state row),
// solves each steady state with GTH (Grassmann-Taksar-Heyman state reduction: subtraction-free,
// so no pivoting is needed; one barrier per eliminated state), and reduces Eq.4-8 and Eq.1.  The CTA that finishes last runs FindCoSchedule's selection (a9):
// per pair argmin dT over its maximal splits, then argmax CP over pairs.
//
// Readings: R1 P_ir = min(1, max(#ready,1)/L); R2 L(n) = L0 + a0 n/B + b0 with n
// the outstanding requests of the idle warps; R3 independent warps (binomial convolution);
// R4/R5 shared round and latency in the joint chain; R14 w = b * wpb / n_sched; R22 guard L > W.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "kl_internal.h"
#include "kl_model_common.cuh"

namespace {

#ifdef KL_MODEL_PROFILE
__device__ __forceinline__ unsigned long long gtimer_m() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif
constexpr int kMaxW = 16;                 // virtual-SM warps (64 warps / 4 schedulers)
constexpr int kMaxS = (kMaxW / 2 + 1) * (kMaxW / 2 + 1);   // 81 joint states at W_v = 16
constexpr int kThreads = 256;

// Binomial coefficients C(n,k), n <= 16 (exact in double).
__constant__ double c_binom[17][17];


// One-kernel transition row from i idle of w (Eq.2 summed with binomial weights, R3), one warp:
// lane a holds Binomial(i, pir) mass at a returns, lane b Binomial(w - i, rm) mass at b stalls;
// lane j returns T(i -> j) = sum_a pA[a] pB[j - i + a] (0 for j > w).  Powers by repeated
// multiplication (no pow()); binomial coefficients from the exact table in shared memory.
__device__ double warp_row(int w, int i, double pir, double rm, const double (*binom)[kMaxW + 1]) {
    const int lane = threadIdx.x & 31, nr = w - i;
    double pa = 0.0, pb = 0.0;
    if (lane <= i) {
        double x = 1.0;
        for (int t = 0; t < lane; ++t) x *= pir;
        for (int t = 0; t < i - lane; ++t) x *= (1.0 - pir);
        pa = binom[i][lane] * x;
    }
    if (lane <= nr) {
        double x = 1.0;
        for (int t = 0; t < lane; ++t) x *= rm;
        for (int t = 0; t < nr - lane; ++t) x *= (1.0 - rm);
        pb = binom[nr][lane] * x;
    }
    double row = 0.0;
    for (int a = 0; a <= i; ++a) {
        const double va = __shfl_sync(0xffffffffu, pa, a);
        const int bb = lane - i + a;
        const double vb = __shfl_sync(0xffffffffu, pb, bb & 31);
        if (bb >= 0 && bb <= nr) row += va * vb;
    }
    return lane <= w ? row : 0.0;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) s += red[i];
    return s;
}

// Steady state and IPCs of the chain of kernel A at wa warps (and kernel B at wb warps; wb = 0,
// kb = null: solo chain).  States (p, q) = idle warps of A and B, S = (wa+1)(wb+1); the row of
// (p, q) is the outer product of the two one-kernel rows under the state's shared round R and
// latency (R4/R5).  The stationary distribution is GTH state reduction (subtraction-
// free) with one barrier per eliminated state on a 16 x 16 thread tile; the threads owning row
// k-1 produce the next pivot sum while updating it.  Returns KL_OK / KL_EINFEASIBLE (guard
// L > W, R22) / KL_ENUMERIC (zero pivot: reducible chain).
struct ChainOut { double ipc_a, ipc_b; };

constexpr int kT = kMaxS / 16 + 1;      // GTH register tile: 6 x 6 doubles per thread

// Publish row k (held in register row M of the owning half-warp): entries j < k to the row
// buffer; returns this thread's part of the pivot sum.  Static M: registers, no local memory.
template <int M>
__device__ __forceinline__ double publish_row(const double (&a)[kT][kT], double* row, int k, int tx) {
    double part = 0.0;
#pragma unroll
    for (int n = 0; n < kT; ++n) {
        const int j = tx + 16 * n;
        const double v = j < k ? a[M][n] : 0.0;
        row[j] = v;
        part += v;
    }
    return part;
}

// Publish column k (register column N of the owning threads), rows i < k, into the back-
// substitution store P[i][k].
template <int N>
__device__ __forceinline__ void publish_col(const double (&a)[kT][kT], double* P, int S, int k, int ty) {
#pragma unroll
    for (int m = 0; m < kT; ++m) {
        const int i = ty + 16 * m;
        if (i < k) P[i * S + k] = a[m][N];
    }
}


__device__ int chain_ipc(const KlModelKind* ka, int wa, const KlModelKind* kb, int wb, const KlModelCfg& c,
                         double* P, double* pi, double* Rs, double* red, const double (*binom)[kMaxW + 1],
                         ChainOut* out) {
    const int nb = wb + 1, S = (wa + 1) * nb;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = kThreads / 32;
    __shared__ int s_bad;
    __shared__ double s_piv[2], s_inv[2];
    __shared__ double inv_s[kMaxS];
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
#ifdef KL_MODEL_PROFILE
    const unsigned long long tq0 = gtimer_m();
#endif
    // ---- chain build: one warp per state row
    for (int s = warp; s < S; s += NW) {
        const int p = s / nb, q = s - p * nb;
        const double R = round_dur(wa - p, ka, wb - q, kb);
        const double n = (double)p * ka->r + (kb ? (double)q * kb->r : 0.0);
        double pr = 0.0;
        if (!p_ir(c, R, p + q, n, &pr)) {
            if (lane == 0) s_bad = KL_EINFEASIBLE;
            continue;
        }
        if (lane == 0) Rs[s] = R;
        const double r1 = warp_row(wa, p, pr, ka->rm, binom);
        const double r2 = kb ? warp_row(wb, q, pr, kb->rm, binom) : (lane == 0 ? 1.0 : 0.0);
        double* row = P + s * S;
        for (int pp = 0; pp <= wa; ++pp) {
            const double v1 = __shfl_sync(0xffffffffu, r1, pp);
            if (lane <= wb) row[pp * nb + lane] = v1 * r2;
        }
    }
    __syncthreads();
    if (s_bad) return s_bad;
#ifdef KL_MODEL_PROFILE
    const unsigned long long tq1 = gtimer_m();
#endif
    // ---- GTH: for k = S-1 .. 1: s_k = sum_{j<k} P[k][j]; P[i][j] += (P[i][k]/s_k) P[k][j], i,j < k.
    // The trailing matrix lives in registers: thread (ty, tx) of a 16 x 16 tile holds
    // a[m][n] = P[ty + 16m][tx + 16n].  Per eliminated state the half-warp owning row k publishes
    // it (and its pivot sum, reduced by shuffles) to a double-buffered row buffer, the threads
    // owning column k publish it into P's column k in shared memory (left unscaled: the back
    // substitution applies 1/s_k and reads exactly these columns), one barrier, then every thread
    // applies the rank-1 update to its registers.  Shared memory carries 2 S values per state
    // instead of the whole k x k update.
    __shared__ double s_row[2][16 * kT];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double a[kT][kT];
#pragma unroll
    for (int m = 0; m < kT; ++m)
#pragma unroll
        for (int n = 0; n < kT; ++n) {
            const int i = ty + 16 * m, j = tx + 16 * n;
            a[m][n] = (i < S && j < S) ? P[i * S + j] : 0.0;
        }
    __syncthreads();   // P is now only the column store for the back substitution
    for (int k = S - 1; k >= 1; --k) {
        const int mk = k >> 4, buf = k & 1;
        if ((ty >> 1) == ((k & 15) >> 1)) {   // the warp holding row k (in one of its halves):
            double part = 0.0;                   // publish the row and its pivot sum
            const bool own = ty == (k & 15);
            if (own) {
                double* row = s_row[buf];
                switch (mk) {
                    case 0: part = publish_row<0>(a, row, k, tx); break;
                    case 1: part = publish_row<1>(a, row, k, tx); break;
                    case 2: part = publish_row<2>(a, row, k, tx); break;
                    case 3: part = publish_row<3>(a, row, k, tx); break;
                    case 4: part = publish_row<4>(a, row, k, tx); break;
                    default: part = publish_row<5>(a, row, k, tx); break;
                }
            }
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            if (own && tx == 0) {
                const double inv = 1.0 / part;
                s_piv[buf] = part;
                s_inv[buf] = inv;
                inv_s[k] = inv;
            }
        }
        if (tx == (k & 15)) {   // threads owning column k: publish it (rows i < k)
            switch (mk) {
                case 0: publish_col<0>(a, P, S, k, ty); break;
                case 1: publish_col<1>(a, P, S, k, ty); break;
                case 2: publish_col<2>(a, P, S, k, ty); break;
                case 3: publish_col<3>(a, P, S, k, ty); break;
                case 4: publish_col<4>(a, P, S, k, ty); break;
                default: publish_col<5>(a, P, S, k, ty); break;
            }
        }
        __syncthreads();
        if (!(s_piv[buf] > 0.0)) return KL_ENUMERIC;   // uniform across the block
        const double inv = s_inv[buf];
        double rk[kT];
#pragma unroll
        for (int n = 0; n < kT; ++n) rk[n] = s_row[buf][tx + 16 * n];   // 0 beyond k
        // rank-1 update over the 16-blocks that hold indices < k (block-uniform bounds: entries
        // of eliminated rows / columns in the last block are dead and may take any update; rows
        // i >= k get c = 0)
        const int kb = (k - 1) >> 4;
#pragma unroll
        for (int m = 0; m < kT; ++m) {
            if (m <= kb) {
                const int i = ty + 16 * m;
                const double c = i < k ? P[i * S + k] * inv : 0.0;
#pragma unroll
                for (int n = 0; n < kT; ++n)
                    if (n <= kb) a[m][n] = fma(c, rk[n], a[m][n]);
            }
        }
    }
    __syncthreads();
#ifdef KL_MODEL_PROFILE
    const unsigned long long tq2 = gtimer_m();
#endif
    // back substitution by warp 0: pi_0 = 1, pi_j = (1/s_j) sum_{i<j} pi_i P[i][j] (column
    // accumulators m = lane + 32 t held in registers)
    if (warp == 0) {
        double acc[3] = {0.0, 0.0, 0.0};
        double tot = 0.0;
        for (int j = 0; j < S; ++j) {
            const int t = j >> 5, src = j & 31;
            const double mine = t == 0 ? acc[0] : (t == 1 ? acc[1] : acc[2]);
            const double pj = j == 0 ? 1.0 : __shfl_sync(0xffffffffu, mine, src) * inv_s[j];
            tot += pj;
            if (lane == 0) pi[j] = pj;
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                const int m = lane + 32 * u;
                if (m > j && m < S) acc[u] = fma(pj, P[j * S + m], acc[u]);
            }
        }
        if (lane == 0) red[8] = tot;
    }
    __syncthreads();
    const double tot = red[8];
#ifdef KL_MODEL_PROFILE
    if (threadIdx.x == 0 && S > 60 && blockIdx.x % 20 == 0) printf("MPC S=%d build %.1f gth %.1f back %.1f us\n", S, (tq1 - tq0) / 1e3, (tq2 - tq1) / 1e3, (gtimer_m() - tq2) / 1e3);
#endif
    double den = 0.0, na = 0.0, nbs = 0.0;
    for (int s = threadIdx.x; s < S; s += kThreads) {
        const int p = s / nb, q = s - p * nb;
        const double g = pi[s] / tot;
        den += g * Rs[s];
        if (p < wa) na += g * (double)(wa - p);
        if (q < wb) nbs += g * (double)(wb - q);
    }
    den = block_sum(den, red);
    na = block_sum(na, red);
    nbs = block_sum(nbs, red);
    out->ipc_a = na / den;
    out->ipc_b = nbs / den;
    __syncthreads();
    return KL_OK;
}

// Grid: cfg.n_cand candidate CTAs, then KL_NKINDS solo CTAs.  Solo CTA kk solves kind kk's solo
// chain at its solo occupancy b^max (Eq.4) once for the whole batch -- every candidate of the
// kind shares it -- into preds[n_cand + kk] (ipc in .solo1); candidate CTAs solve only their
// joint chain (Eq.5-7).  The CTA that finishes last completes every prediction (solo IPCs, Eq.1
// CP, Eq.8 dT), publishes them, and runs the selection (a9) if n_pairs > 0.
__global__ void __launch_bounds__(kThreads, 2)   // 2 CTAs per SM: a 202-candidate batch stays one wave
k_model_batch(const KlModelKind* __restrict__ kinds, const KlModelCfg cfg, const KlCand* __restrict__ cands,
              kl_prediction* preds, int n_pairs, const int32_t* __restrict__ pair_off,
              uint32_t* done_counter, KlDecision* dec) {
    extern __shared__ __align__(16) double smem_d[];
    double* P = smem_d;                    // kMaxS * kMaxS
    double* pi = P + kMaxS * kMaxS;        // kMaxS
    double* Rs = pi + kMaxS;               // kMaxS
    double* red = Rs + kMaxS;              // 16
    __shared__ double s_binom[kMaxW + 1][kMaxW + 1];
    __shared__ KlCand s_cd;
    __shared__ KlModelKind s_kall[KL_NKINDS];
    const int n = cfg.n_cand;
    const bool solo_cta = (int)blockIdx.x >= n;
    for (int x = threadIdx.x; x < (kMaxW + 1) * (kMaxW + 1); x += kThreads)
        s_binom[x / (kMaxW + 1)][x % (kMaxW + 1)] = c_binom[x / (kMaxW + 1)][x % (kMaxW + 1)];
    // the host-mapped inputs in ONE PCIe round trip: the kind table as 8-byte words, one per
    // thread, and this CTA's candidate by another warp, in parallel (a dependent cand -> kinds
    // read by one thread held the whole CTA at this barrier for ~20 % of the batch's warp time)
    static_assert(sizeof(KlModelKind) % 8 == 0, "kind table copied as 8-byte words");
    constexpr int kKindWords = KL_NKINDS * (int)sizeof(KlModelKind) / 8;
    static_assert(kKindWords < kThreads - 32, "kind table fits the first warps");
    if ((int)threadIdx.x < kKindWords)
        reinterpret_cast<unsigned long long*>(s_kall)[threadIdx.x] =
            reinterpret_cast<const unsigned long long*>(kinds)[threadIdx.x];
    if (threadIdx.x == kThreads - 1 && !solo_cta) s_cd = cands[blockIdx.x];
    __syncthreads();
#ifdef KL_MODEL_PROFILE
    unsigned long long tp0 = gtimer_m();
#endif
    ChainOut co;
    if (solo_cta) {
        const KlModelKind k1 = s_kall[blockIdx.x - n];
        const int ts = k1.bsolo * k1.wpb, ws = ts / cfg.n_sched;
        int status = (ts % cfg.n_sched || ws < 1 || ws > cfg.W || cfg.W > kMaxW) ? KL_EINFEASIBLE : 0;
        if (status == 0) {
            status = chain_ipc(&k1, ws, nullptr, 0, cfg, P, pi, Rs, red, s_binom, &co);
            if (status == KL_EINFEASIBLE) status = KL_ENUMERIC;
        }
        if (threadIdx.x == 0) {
            kl_prediction o = {};
            o.solo1 = status == 0 ? co.ipc_a : 0.0;
            o.status = status;
            preds[blockIdx.x] = o;
        }
    } else {
        const KlCand cd = s_cd;
        const KlModelKind k1 = s_kall[cd.k1], k2 = s_kall[cd.k2];
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
        if (status == 0) {   // joint chain, Eq.5-7 with R_(i,j) = joint round duration (R4)
            status = chain_ipc(&k1, w1, solo_query ? nullptr : &k2, solo_query ? 0 : w2, cfg, P, pi, Rs, red,
                               s_binom, &co);
            if (status == KL_EINFEASIBLE) status = KL_ENUMERIC;
            if (status == 0) {
                out.ipc1 = co.ipc_a;
                out.ipc2 = co.ipc_b;
                out.c = out.ipc1 + out.ipc2;
            }
        }
        out.status = status;
        if (threadIdx.x == 0) {
            preds[blockIdx.x] = out;
            if (cfg.cands_dev) cfg.cands_dev[blockIdx.x] = cd;
        }
    }
#ifdef KL_MODEL_PROFILE
    if (threadIdx.x == 0 && blockIdx.x % 20 == 0)
        printf("MP cta %d %s chain %.1f us\n", blockIdx.x, solo_cta ? "solo" : "joint", (gtimer_m() - tp0) / 1e3);
#endif
    if (!last_cta(done_counter)) return;
    // the last CTA: complete every prediction with the shared solo IPCs (Eq.4), Eq.1 and Eq.8
    const KlCand* cl = cfg.cands_dev ? cfg.cands_dev : cands;
    for (int i = threadIdx.x; i < n; i += kThreads) {
        kl_prediction o = preds[i];
        const KlCand cd = cl[i];
        if (o.status != KL_EINFEASIBLE) {
            const kl_prediction s1 = preds[n + cd.k1], s2 = preds[n + cd.k2];
            if (s1.status || s2.status) {
                o.status = KL_ENUMERIC;   // a solo chain failed (range failures are caught above)
            } else {
                o.solo1 = s1.solo1;
                o.solo2 = s2.solo1;
                if (o.status == 0 && cd.b2 != 0) {
                    o.cp = 1.0 - 1.0 / (o.ipc1 / o.solo1 + o.ipc2 / o.solo2);   // Eq.1
                    o.dT = fabs(s_kall[cd.k1].ipb * (double)cd.b1 / o.ipc1 -
                                s_kall[cd.k2].ipb * (double)cd.b2 / o.ipc2);      // Eq.8
                }
            }
        }
        preds[i] = o;
        if (cfg.preds_host) cfg.preds_host[i] = o;   // the host reads these (mapped)
    }
    __threadfence();
    __syncthreads();
    if (n_pairs > 0) {
        select_body<kThreads>(cfg, s_kall, cl, preds, n_pairs, pair_off, done_counter, dec);
    } else if (threadIdx.x == 0) {
        *done_counter = 0u;
    }
}

}  // namespace

// One-time setup, called by kl_create (eager: a lazily loaded kernel or a symbol copy during
// scheduling would synchronise the device behind unrelated streams).
int kl_dev_model_init() {
    const size_t smem = sizeof(double) * (kMaxS * kMaxS + 2 * kMaxS + 16);
    cudaError_t e = cudaFuncSetAttribute(k_model_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    double tab[17][17] = {};
    for (int n = 0; n <= 16; ++n) {
        tab[n][0] = 1.0;
        for (int k = 1; k <= n; ++k) tab[n][k] = tab[n - 1][k - 1] + (k <= n - 1 ? tab[n - 1][k] : 0.0);
    }
    e = cudaMemcpyToSymbol(c_binom, tab, sizeof(tab));
    if (e != cudaSuccess) return (int)e;
    cudaFuncAttributes fa;
    return (int)cudaFuncGetAttributes(&fa, k_model_batch);
}

int kl_dev_model_batch(const KlModelKind* kinds, KlModelCfg cfg, const KlCand* cands,
                       kl_prediction* preds, int n_pairs, const int32_t* pair_off,
                       uint32_t* done_counter, KlDecision* dec, void* stream) {
    if (cfg.n_cand <= 0) return 0;
    const size_t smem = sizeof(double) * (kMaxS * kMaxS + 2 * kMaxS + 16);
    static bool attr = false;
    if (!attr) {
        int e = kl_dev_model_init();
        if (e) return e;
        attr = true;
    }
    k_model_batch<<<cfg.n_cand + KL_NKINDS, kThreads, smem, (cudaStream_t)stream>>>(kinds, cfg, cands, preds, n_pairs,
                                                                      pair_off, done_counter, dec);
    return (int)cudaGetLastError();
}
