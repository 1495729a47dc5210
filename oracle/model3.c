/* model3.c -- f1: the three-state (coalesced / uncoalesced) extension of the warp-state model
 * (TEST INFRASTRUCTURE; plain fp64, dense LU from model.c; no code shared with the CUDA path).
 *
 * PAPER.md P:1000-1019 ("Uncoalesced Access"): a warp is ready, stalled on a coalesced access or
 * stalled on an uncoalesced access (labels as in reading R12); uncoalesced accesses generate more
 * memory traffic, so their latency is higher; both latencies follow the linear model; the ratio of
 * coalesced to uncoalesced memory instructions extends the two-state transitions.  Readings
 * (R27):
 *   - per kind: Rm (memory instruction ratio), uc (fraction of memory instructions that are
 *     uncoalesced), r (requests per coalesced memory instruction), ru (per uncoalesced one);
 *   - a ready warp stalls coalesced w.p. Rm(1-uc), uncoalesced w.p. Rm*uc (else stays ready);
 *     a coalesced-idle warp returns w.p. P_c = min(1, R/L_c), an uncoalesced-idle one w.p.
 *     P_u = min(1, R/L_u); warps move independently (R3), so one kernel's row is a binomial
 *     (returns of each idle class) times a multinomial (new stalls of the ready warps);
 *   - outstanding requests n = sum_k (c_k r_k + u_k ru_k); L_c(n) = L0 + a0 n/B + b0 exactly as
 *     the two-state model (R2); L_u = L_c + a0 (ru - r)/B: the extra requests of an uncoalesced
 *     instruction queue at the virtual SM's bandwidth B;
 *   - the round duration and the pipe ceilings are the two-state ones (R1, R4, R26) over the
 *     ready warps; the joint chain is the product of the two kernels' rows under the shared
 *     round and latency (R5); IPC as Eq.4-7 with R_(i,j) the round duration.
 * With uc = 0 (or ru = r) the chain reduces exactly to the two-state chain (pinned).
 *
 * Block granularity ("consider the thread block as a scheduling unit", reading R13):
 * a kernel may be modelled in units of g warps that move together (g = the block's warps per
 * virtual SM); w then counts units, a ready unit issues g instructions per round (the round and
 * the pipe ceilings see g x ready warps), an idle unit keeps g x r (g x ru) requests outstanding,
 * and IPC counts g instructions per ready unit.  g = 1 is the warp model.
 *
 * One kernel's state (c, u): c coalesced-idle, u uncoalesced-idle warps, c + u <= w; index
 * idx(c, u) = sum_{c'<c} (w - c' + 1) + u.  Joint state (s1, s2) -> s1 * n2 + s2.
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

static double binom3(int n, int k) {
    if (k < 0 || k > n) return 0.0;
    double r = 1.0;
    for (int i = 1; i <= k; ++i) r = r * (double)(n - k + i) / (double)i;
    return r;
}

int or3_nstates(int w) { return (w + 1) * (w + 2) / 2; }

static int idx3(int w, int c, int u) { return c * (w + 1) - c * (c - 1) / 2 + u; }

static double pipe3(const or_kmodel3* k) { return (k->pi > 0.0 && k->pi < 1.0) ? k->pi : 1.0; }

/* Round duration, as model.c round_of (R1, R26). */
static double round3(int ready1, const or_kmodel3* k1, int ready2, const or_kmodel3* k2) {
    const double p1 = k1 ? pipe3(k1) : 1.0, p2 = k2 ? pipe3(k2) : 1.0;
    double R = (double)(ready1 + ready2);
    if (k1 && k2 && k1->pipe != 0 && k1->pipe == k2->pipe) {
        double t = ready1 / p1 + ready2 / p2;
        if (t > R) R = t;
    } else {
        if (ready1 / p1 > R) R = ready1 / p1;
        if (ready2 / p2 > R) R = ready2 / p2;
    }
    return R > 1.0 ? R : 1.0;
}

/* Row of one kernel from (c, u) over its or3_nstates(w) states, for return probabilities pc, pu. */
void or3_row(const or_kmodel3* k, int w, int c, int u, double pc, double pu, double* row) {
    const int n = or3_nstates(w), ready = w - c - u;
    const double sc = k->rm * (1.0 - k->uc), su = k->rm * k->uc, st = 1.0 - k->rm;
    for (int j = 0; j < n; ++j) row[j] = 0.0;
    for (int a = 0; a <= c; ++a) {                       /* coalesced-idle warps that return */
        const double pa = binom3(c, a) * pow(pc, a) * pow(1.0 - pc, c - a);
        for (int b = 0; b <= u; ++b) {                   /* uncoalesced-idle warps that return */
            const double pb = binom3(u, b) * pow(pu, b) * pow(1.0 - pu, u - b);
            for (int x = 0; x <= ready; ++x)             /* ready warps that stall coalesced */
                for (int y = 0; x + y <= ready; ++y) {   /* ... and uncoalesced */
                    const double px = binom3(ready, x) * binom3(ready - x, y) * pow(sc, x) * pow(su, y) *
                                      pow(st, ready - x - y);
                    row[idx3(w, c - a + x, u - b + y)] += pa * pb * px;
                }
        }
    }
}

/* Latencies of the two access classes of kernel k given the outstanding requests n. */
static int lat3(const or_smcfg* cfg, const or_kmodel3* k, double R, int idle, double n, double* pc, double* pu) {
    const double Lc = or_latency(cfg, n, idle);
    if (!(Lc > (double)cfg->W)) return -1;               /* guard R22 */
    const double Lu = Lc + cfg->a0 * (k->ru - k->r) / cfg->B;
    const double a = R / Lc, b = R / Lu;
    *pc = a < 1.0 ? a : 1.0;
    *pu = b < 1.0 ? b : 1.0;
    return 0;
}

/* Joint (or, with k2 = NULL / w2 = 0, solo) three-state chain: P is S x S, R the round
 * duration of every state, S = or3_nstates(w1) * or3_nstates(w2). */
int or3_build(const or_kmodel3* k1, int w1, const or_kmodel3* k2, int w2, const or_smcfg* cfg, double* P,
              double* R) {
    const int n1 = or3_nstates(w1), n2 = k2 ? or3_nstates(w2) : 1, S = n1 * n2;
    const int g1 = k1->g > 0 ? k1->g : 1, g2 = (k2 && k2->g > 0) ? k2->g : 1;
    double* r1 = (double*)malloc(sizeof(double) * n1);
    double* r2 = (double*)malloc(sizeof(double) * n2);
    int rc = 0;
    for (int c1 = 0; c1 <= w1 && !rc; ++c1)
        for (int u1 = 0; c1 + u1 <= w1 && !rc; ++u1)
            for (int c2 = 0; c2 <= (k2 ? w2 : 0) && !rc; ++c2)
                for (int u2 = 0; c2 + u2 <= (k2 ? w2 : 0) && !rc; ++u2) {
                    const int s = idx3(w1, c1, u1) * n2 + (k2 ? idx3(w2, c2, u2) : 0);
                    const int rd1 = w1 - c1 - u1, rd2 = k2 ? w2 - c2 - u2 : 0;
                    R[s] = round3(g1 * rd1, k1, g2 * rd2, k2);
                    const int idle = g1 * (c1 + u1) + g2 * (c2 + u2);
                    const double n = g1 * (c1 * k1->r + u1 * k1->ru) + (k2 ? g2 * (c2 * k2->r + u2 * k2->ru) : 0.0);
                    double pc1, pu1, pc2 = 0.0, pu2 = 0.0;
                    if (lat3(cfg, k1, R[s], idle, n, &pc1, &pu1) ||
                        (k2 && lat3(cfg, k2, R[s], idle, n, &pc2, &pu2))) {
                        rc = -1;
                        break;
                    }
                    or3_row(k1, w1, c1, u1, pc1, pu1, r1);
                    if (k2) or3_row(k2, w2, c2, u2, pc2, pu2, r2);
                    else r2[0] = 1.0;
                    for (int t1 = 0; t1 < n1; ++t1)
                        for (int t2 = 0; t2 < n2; ++t2) P[(size_t)s * S + t1 * n2 + t2] = r1[t1] * r2[t2];
                }
    free(r1);
    free(r2);
    return rc;
}

/* Eq.4-7 over the three-state chain: issued instructions (ready warps) over elapsed cycles. */
void or3_ipc(int w1, int w2, int joint, const double* pi, const double* R, double* ipc1, double* ipc2) {
    or3_ipc_g(w1, 1, w2, 1, joint, pi, R, ipc1, ipc2);
}

/* Eq.4-7 with units of g warps: a ready unit issues g instructions per round. */
void or3_ipc_g(int w1, int g1, int w2, int g2, int joint, const double* pi, const double* R, double* ipc1,
               double* ipc2) {
    const int n2 = joint ? or3_nstates(w2) : 1;
    double den = 0.0, a = 0.0, b = 0.0;
    for (int c1 = 0; c1 <= w1; ++c1)
        for (int u1 = 0; c1 + u1 <= w1; ++u1)
            for (int c2 = 0; c2 <= (joint ? w2 : 0); ++c2)
                for (int u2 = 0; c2 + u2 <= (joint ? w2 : 0); ++u2) {
                    const int s = idx3(w1, c1, u1) * n2 + (joint ? idx3(w2, c2, u2) : 0);
                    den += pi[s] * R[s];
                    a += pi[s] * (double)(w1 - c1 - u1);
                    if (joint) b += pi[s] * (double)(w2 - c2 - u2);
                }
    *ipc1 = g1 * a / den;
    *ipc2 = joint ? g2 * b / den : 0.0;
}

/* Units of a kernel on the virtual SM: b blocks of wpb warps over nsched schedulers, in units of
 * g warps (R14, R13); -1 if not whole. */
static int vsm3(const or_kmodel3* k, int b, int nsched) {
    const int t = b * k->wpb, g = k->g > 0 ? k->g : 1;
    if (t % nsched) return -1;
    const int w = t / nsched;
    return (w % g) ? -1 : w / g;
}
static int gof(const or_kmodel3* k) { return k->g > 0 ? k->g : 1; }

double or3_solo_ipc(const or_kmodel3* k, int b, int nsched, const or_smcfg* cfg, int* status) {
    const int w = vsm3(k, b, nsched);
    *status = 0;
    if (w < 1 || w * gof(k) > cfg->W) { *status = 2; return 0.0; }
    const int S = or3_nstates(w);
    double* P = (double*)malloc(sizeof(double) * (size_t)S * S);
    double* R = (double*)malloc(sizeof(double) * S);
    double* pi = (double*)malloc(sizeof(double) * S);
    double ipc = 0.0, dummy;
    if (or3_build(k, w, 0, 0, cfg, P, R) || or_stationary(S, P, pi)) *status = 6;
    else or3_ipc_g(w, gof(k), 0, 1, 0, pi, R, &ipc, &dummy);
    free(P); free(R); free(pi);
    return ipc;
}

void or3_predict(const or_kmodel3* k1, int b1, int b1max, const or_kmodel3* k2, int b2, int b2max, int nsched,
                 const or_smcfg* cfg, or_pred* out) {
    memset(out, 0, sizeof(*out));
    const int w1 = vsm3(k1, b1, nsched), w2 = vsm3(k2, b2, nsched);
    if (w1 < 1 || w2 < 1 || w1 * gof(k1) + w2 * gof(k2) > cfg->W) { out->status = 2; return; }
    int st1, st2;
    out->solo1 = or3_solo_ipc(k1, b1max, nsched, cfg, &st1);
    out->solo2 = or3_solo_ipc(k2, b2max, nsched, cfg, &st2);
    if (st1 || st2) { out->status = st1 ? st1 : st2; return; }
    const int S = or3_nstates(w1) * or3_nstates(w2);
    double* P = (double*)malloc(sizeof(double) * (size_t)S * S);
    double* R = (double*)malloc(sizeof(double) * S);
    double* pi = (double*)malloc(sizeof(double) * S);
    if (or3_build(k1, w1, k2, w2, cfg, P, R) || or_stationary(S, P, pi)) {
        out->status = 6;
    } else {
        or3_ipc_g(w1, gof(k1), w2, gof(k2), 1, pi, R, &out->ipc1, &out->ipc2);
        out->c = out->ipc1 + out->ipc2;
        double cipc[2] = {out->ipc1, out->ipc2}, ipc[2] = {out->solo1, out->solo2};
        out->cp = or_cp(2, cipc, ipc);
        out->dT = fabs(k1->ipb * b1 / out->ipc1 - k2->ipb * b2 / out->ipc2);   /* Eq.8 */
    }
    free(P); free(R); free(pi);
}
