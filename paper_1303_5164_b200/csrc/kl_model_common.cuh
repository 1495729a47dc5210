// kl_model_common.cuh -- device helpers shared by the model kernels (kl_model.cu: two-state
// warp model in shared memory; kl_model3.cu: three-state / block-granularity model): the round,
// the latency model, the split order and the fused FindCoSchedule selection (a9).  Product path.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "kl_internal.h"

namespace {

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

__device__ __forceinline__ double band(double x, double y) {
    double m = fmax(1.0, fmax(fabs(x), fabs(y)));
    return 1e-12 * m;
}

// a9 split order: argmin dT; ties (1e-12 band): larger C, more warps, smaller b1.
// Eq.8 time scale of a split: the larger of its two per-wave times I_k b_k / cIPC_k; dT ties are
// judged relative to it (R8: dT is a difference of such terms, so its rounding noise scales
// with them, not with dT).
__device__ __forceinline__ double dT_scale(const kl_prediction& p, const KlCand& c, const KlModelKind* kinds) {
    return fmax(kinds[c.k1].ipb * (double)c.b1 / p.ipc1, kinds[c.k2].ipb * (double)c.b2 / p.ipc2);
}

// a9 split order: argmin dT (ties within 1e-9 of the Eq.8 terms); then larger C (1e-12 band),
// more warps, smaller b1.  rule 1: highest predicted CP first (R7').
__device__ bool better_split(const kl_prediction& a, const KlCand& ca, const kl_prediction& b, const KlCand& cb,
                             int rule, const KlModelKind* kinds) {
    if (rule == 1) {   // ablation: highest predicted CP first
        double t = band(a.cp, b.cp);
        if (a.cp > b.cp + t) return true;
        if (a.cp < b.cp - t) return false;
    }
    double t = 1e-9 * fmax(dT_scale(a, ca, kinds), dT_scale(b, cb, kinds));
    if (a.dT < b.dT - t) return true;
    if (a.dT > b.dT + t) return false;
    t = band(a.c, b.c);
    if (a.c > b.c + t) return true;
    if (a.c < b.c - t) return false;
    if (ca.warps != cb.warps) return ca.warps > cb.warps;
    return ca.b1 < cb.b1;
}

// True in every thread of the CTA that finishes last (the others see false); each CTA calls it
// once after writing its prediction.  The last CTA resets the counter in select_body (or itself
// when no selection follows).
__device__ __forceinline__ bool last_cta(uint32_t* done_counter) {
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(done_counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (s_last) __threadfence();
    return s_last != 0;
}

// Fused selection (a9) by the CTA that finishes last: per pair the best split (better_split),
// then argmax CP over pairs.  Called by every CTA after writing its prediction.
template <int kThreads>
__device__ void select_body(const KlModelCfg& cfg, const KlModelKind* kinds_in, const KlCand* __restrict__ cands,
                            const kl_prediction* preds, int n_pairs, const int32_t* __restrict__ pair_off,
                            uint32_t* done_counter, KlDecision* dec) {
    __shared__ int s_best_pair[128];
    __shared__ KlModelKind kinds[KL_NKINDS];   // staged: the table lives in host-mapped memory
    for (int k = threadIdx.x; k < KL_NKINDS; k += kThreads) kinds[k] = kinds_in[k];
    __syncthreads();
    for (int pr = threadIdx.x; pr < n_pairs; pr += kThreads) {
        int best = -1;
        kl_prediction bp;
        KlCand bc;
        for (int i = pair_off[pr]; i < pair_off[pr + 1]; ++i) {
            kl_prediction a = preds[i];
            if (a.status != 0) continue;
            KlCand ca = cands[i];
            if (best < 0 || better_split(a, ca, bp, bc, cfg.split_rule, kinds)) { best = i; bp = a; bc = ca; }
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

template <int kThreads>
__device__ void select_last(const KlModelCfg& cfg, const KlModelKind* kinds, const KlCand* __restrict__ cands,
                            const kl_prediction* preds, int n_pairs, const int32_t* __restrict__ pair_off,
                            uint32_t* done_counter, KlDecision* dec) {
    if (last_cta(done_counter)) select_body<kThreads>(cfg, kinds, cands, preds, n_pairs, pair_off, done_counter, dec);
}

}  // namespace
