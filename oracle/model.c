/* model.c -- O2/O3: the paper's Markov-chain warp-state model, occupancy and pruning
 * (TEST INFRASTRUCTURE; plain fp64, dense LU; no code shared with the CUDA path).
 *
 * The model is an approximation, so this file follows the algorithm step by step in the order
 * and notation of PAPER.md §4.4:
 *   per-warp probabilities  ->  round as time step
 *   -> linear latency model (reading R2) -> Eq.2 transitions (R3)
 *   -> steady state Eq.3 -> IPC Eq.4
 *   -> heterogeneous chain (R5) -> Eq.5-7 (R4) -> CP Eq.1
 *   -> balanced slice ratio Eq.8, on the virtual SM of P:1023-1036 (R14).
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Latency L as a function of the outstanding memory requests n (reading R2 of the garbled
 * "L = L0 + B/(a0 S_i) + b0"): linear contention L0 + a0*n/B + b0.  Mode 1 keeps the
 * verbatim expression with S_i read as the idle-warp count. */
double or_latency(const or_smcfg* c, double n, int idle) {
    if (c->latency_mode == 1) return c->L0 + c->B / (c->a0 * (idle > 1 ? idle : 1)) + c->b0;
    return c->L0 + c->a0 * n / c->B + c->b0;
}

static double binom(int n, int k) {
    if (k < 0 || k > n) return 0.0;
    double r = 1.0;
    for (int i = 1; i <= k; ++i) r = r * (double)(n - k + i) / (double)i;
    return r;
}

/* Row i of one kernel's idle-count chain (Eq.2): from S_i, N_ir = a of the i idle
 * warps become ready (each with p_ir) and N_ri = b of the w-i ready warps become idle (each
 * with Rm); S_j = S_i - a + b.  Distinct (a,b) are mutually exclusive events, so their
 * probabilities add; warps move independently (R3). */
void or_row(int w, int i, double p_ir, double rm, double* row) {
    for (int j = 0; j <= w; ++j) row[j] = 0.0;
    for (int a = 0; a <= i; ++a) {
        double pa = binom(i, a) * pow(p_ir, a) * pow(1.0 - p_ir, i - a);
        for (int b = 0; b <= w - i; ++b) {
            double pb = binom(w - i, b) * pow(rm, b) * pow(1.0 - rm, w - i - b);
            row[i - a + b] += pa * pb;
        }
    }
}

/* Pipe ceiling of a kernel (R26); 0 means 1 (the paper's issue-only model). */
static double pipe_of(const or_kmodel* k) { return (k->pi > 0.0 && k->pi < 1.0) ? k->pi : 1.0; }

/* Round duration: every ready warp issues one instruction, so a round
 * lasts #ready cycles, or 1 if none is ready (R1).  B200 adaptation R26: a kernel whose busiest
 * pipe sustains only pi instructions per cycle needs ready/pi cycles of that pipe; kernels on the
 * same pipe share it (their pipe times add), kernels on different pipes overlap.  The round lasts
 * until the slowest of (issue of all ready warps, every pipe) is done; pi = 1 for every kernel
 * gives back the paper's max(#ready, 1) exactly. */
static double round_of(int ready1, const or_kmodel* k1, int ready2, const or_kmodel* k2) {
    const double p1 = k1 ? pipe_of(k1) : 1.0, p2 = k2 ? pipe_of(k2) : 1.0;
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

/* P_{i->r} in a state with round duration R, `idle` idle warps and n outstanding requests: the
 * literal (W-I)/L with (W-I) the round duration (R1), clamped to 1 when the round
 * outlasts the latency. */
static int p_idle_to_ready(const or_smcfg* c, double R, int idle, double n, double* out) {
    if (c->pir_mode == 1) { *out = c->const_q; return 0; }
    double L = or_latency(c, n, idle);
    if (!(L > (double)c->W)) return -1;            /* guard R22: reducible chain otherwise */
    double p = R / L;
    *out = p < 1.0 ? p : 1.0;
    return 0;
}

int or_build_homog(const or_kmodel* k, int w, const or_smcfg* c, double* P, double* R) {
    for (int i = 0; i <= w; ++i) {
        int ready = w - i;
        double p_ir;
        R[i] = round_of(ready, k, 0, 0);               /* round duration, P:910-914 (+R26) */
        if (p_idle_to_ready(c, R[i], i, (double)i * k->r, &p_ir)) return -1;
        or_row(w, i, p_ir, k->rm, &P[(size_t)i * (w + 1)]);
    }
    return 0;
}

/* Heterogeneous chain: state (p,q) = idle warps of K1, K2.  Both kernels share the
 * round (R = total ready warps) and the memory system (L over all outstanding
 * requests); given the state, the kernels move independently, so the transition probability is
 * the product of the two single-kernel rows. */
int or_build_joint(const or_kmodel* k1, int w1, const or_kmodel* k2, int w2,
                   const or_smcfg* c, double* P, double* R) {
    int S = (w1 + 1) * (w2 + 1);
    double* r1 = (double*)malloc(sizeof(double) * (w1 + 1));
    double* r2 = (double*)malloc(sizeof(double) * (w2 + 1));
    for (int p = 0; p <= w1; ++p)
        for (int q = 0; q <= w2; ++q) {
            int s = p * (w2 + 1) + q;
            double p_ir;
            R[s] = round_of(w1 - p, k1, w2 - q, k2);
            if (p_idle_to_ready(c, R[s], p + q, (double)p * k1->r + (double)q * k2->r, &p_ir)) {
                free(r1); free(r2);
                return -1;
            }
            or_row(w1, p, p_ir, k1->rm, r1);
            or_row(w2, q, p_ir, k2->rm, r2);
            for (int pp = 0; pp <= w1; ++pp)
                for (int qq = 0; qq <= w2; ++qq)
                    P[(size_t)s * S + pp * (w2 + 1) + qq] = r1[pp] * r2[qq];
        }
    free(r1); free(r2);
    return 0;
}

/* Steady state (Eq.3): the left eigenvector of P for eigenvalue one, i.e. the solution
 * of (P^T - I) pi = 0 normalised by sum(pi) = 1 (last equation replaced).  Dense Gaussian
 * elimination with partial pivoting, then back substitution. */
int or_stationary(int S, const double* P, double* pi) {
    double* A = (double*)malloc(sizeof(double) * (size_t)S * S);
    double* b = (double*)malloc(sizeof(double) * S);
    for (int i = 0; i < S; ++i) {
        for (int j = 0; j < S; ++j) A[(size_t)i * S + j] = P[(size_t)j * S + i] - (i == j ? 1.0 : 0.0);
        b[i] = 0.0;
    }
    for (int j = 0; j < S; ++j) A[(size_t)(S - 1) * S + j] = 1.0;
    b[S - 1] = 1.0;
    int rc = 0;
    for (int col = 0; col < S; ++col) {
        int piv = col;
        for (int r = col + 1; r < S; ++r)
            if (fabs(A[(size_t)r * S + col]) > fabs(A[(size_t)piv * S + col])) piv = r;
        if (fabs(A[(size_t)piv * S + col]) < 1e-300) { rc = -1; break; }
        if (piv != col) {
            for (int j = 0; j < S; ++j) {
                double t = A[(size_t)col * S + j];
                A[(size_t)col * S + j] = A[(size_t)piv * S + j];
                A[(size_t)piv * S + j] = t;
            }
            double t = b[col]; b[col] = b[piv]; b[piv] = t;
        }
        for (int r = col + 1; r < S; ++r) {
            double f = A[(size_t)r * S + col] / A[(size_t)col * S + col];
            if (f == 0.0) continue;
            for (int j = col; j < S; ++j) A[(size_t)r * S + j] -= f * A[(size_t)col * S + j];
            b[r] -= f * b[col];
        }
    }
    if (rc == 0)
        for (int i = S - 1; i >= 0; --i) {
            double s = b[i];
            for (int j = i + 1; j < S; ++j) s -= A[(size_t)i * S + j] * pi[j];
            pi[i] = s / A[(size_t)i * S + i];
        }
    free(A); free(b);
    return rc;
}

/* Eq.4: IPC = sum_{i<W} g_i (W-i) / (sum_{i<W} g_i (W-i) + g_W), i.e. issued
 * instructions over elapsed cycles; with the round durations R_i of the chain (R26) the
 * denominator is sum_i g_i R_i (identical to Eq.4 when every R_i = max(W-i, 1)). */
double or_ipc_homog_r(int w, const double* pi, const double* R) {
    double num = 0.0, den = 0.0;
    for (int i = 0; i <= w; ++i) {
        if (i < w) num += pi[i] * (double)(w - i);
        den += pi[i] * R[i];
    }
    return num / den;
}

double or_ipc_homog(int w, const double* pi) {
    double num = 0.0;
    for (int i = 0; i < w; ++i) num += pi[i] * (double)(w - i);
    return num / (num + pi[w]);
}

/* Eq.5-7, R_(i,j) read as the joint round duration (R4). */
void or_ipc_joint(int w1, int w2, const double* pi, const double* R,
                  double* ipc1, double* ipc2, double* c) {
    double den = 0.0, n1 = 0.0, n2 = 0.0;
    for (int p = 0; p <= w1; ++p)
        for (int q = 0; q <= w2; ++q) {
            int s = p * (w2 + 1) + q;
            den += pi[s] * R[s];
            if (p < w1) n1 += pi[s] * (double)(w1 - p);
            if (q < w2) n2 += pi[s] * (double)(w2 - q);
        }
    *ipc1 = n1 / den;
    *ipc2 = n2 / den;
    *c = *ipc1 + *ipc2;
}

/* Eq.1: CP = 1 - 1 / sum_i cIPC_i / IPC_i. */
double or_cp(int n, const double* cipc, const double* ipc) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += cipc[i] / ipc[i];
    return 1.0 - 1.0 / s;
}

/* Warps of a kernel on the virtual SM (R14): b blocks per SM of wpb warps, split
 * over nsched schedulers.  -1 if not a whole number of warps. */
static int vsm_warps(const or_kmodel* k, int b, int nsched) {
    int t = b * k->wpb;
    return (t % nsched) ? -1 : t / nsched;
}

double or_solo_ipc(const or_kmodel* k, int b, int nsched, const or_smcfg* c, int* status) {
    int w = vsm_warps(k, b, nsched);
    *status = 0;
    if (w < 1 || w > c->W) { *status = 2; return 0.0; }
    int S = w + 1;
    double* P = (double*)malloc(sizeof(double) * S * S);
    double* R = (double*)malloc(sizeof(double) * S);
    double* pi = (double*)malloc(sizeof(double) * S);
    double ipc = 0.0;
    if (or_build_homog(k, w, c, P, R) || or_stationary(S, P, pi)) *status = 6;
    else ipc = or_ipc_homog_r(w, pi, R);
    free(P); free(R); free(pi);
    return ipc;
}

void or_predict(const or_kmodel* k1, int b1, int b1max, const or_kmodel* k2, int b2, int b2max,
                int nsched, const or_smcfg* c, or_pred* out) {
    memset(out, 0, sizeof(*out));
    int w1 = vsm_warps(k1, b1, nsched), w2 = vsm_warps(k2, b2, nsched);
    if (w1 < 1 || w2 < 1 || w1 + w2 > c->W) { out->status = 2; return; }
    int st1, st2;
    out->solo1 = or_solo_ipc(k1, b1max, nsched, c, &st1);
    out->solo2 = or_solo_ipc(k2, b2max, nsched, c, &st2);
    if (st1 || st2) { out->status = st1 ? st1 : st2; return; }
    int S = (w1 + 1) * (w2 + 1);
    double* P = (double*)malloc(sizeof(double) * (size_t)S * S);
    double* R = (double*)malloc(sizeof(double) * S);
    double* pi = (double*)malloc(sizeof(double) * S);
    if (or_build_joint(k1, w1, k2, w2, c, P, R) || or_stationary(S, P, pi)) {
        out->status = 6;
    } else {
        or_ipc_joint(w1, w2, pi, R, &out->ipc1, &out->ipc2, &out->c);
        double cipc[2] = {out->ipc1, out->ipc2}, ipc[2] = {out->solo1, out->solo2};
        out->cp = or_cp(2, cipc, ipc);
        /* Eq.8 per wave of b_i blocks per SM: |I1 P1/IPC1 - I2 P2/IPC2| */
        out->dT = fabs(k1->ipb * b1 / out->ipc1 - k2->ipb * b2 / out->ipc2);
    }
    free(P); free(R); free(pi);
}

/* Occupancy: co-resident blocks must fit every per-SM resource.  Registers are
 * allocated per warp in units of reg_unit registers; each block also reserves 1 KiB of shared
 * memory on sm_90+ (CUDA occupancy rules); TMEM columns per block as allocated. */
int or_fits(const or_smres* sm, const or_kres* k1, int b1, const or_kres* k2, int b2) {
    const or_kres* ks[2] = {k1, k2};
    int bs[2] = {b1, b2};
    long warps = 0, blocks = 0, regs = 0, smem = 0, tmem = 0;
    for (int i = 0; i < 2; ++i) {
        if (!ks[i] || bs[i] == 0) continue;
        long rw = ((long)ks[i]->regs * 32 + sm->reg_unit - 1) / sm->reg_unit * sm->reg_unit;
        warps += (long)bs[i] * ks[i]->wpb;
        blocks += bs[i];
        regs += (long)bs[i] * ks[i]->wpb * rw;
        smem += (long)bs[i] * (ks[i]->smem + 1024);
        tmem += (long)bs[i] * ks[i]->tmem;
    }
    if (warps > sm->max_warps) return 1;
    if (blocks > sm->max_blocks) return 2;
    if (regs > sm->max_regs) return 3;
    if (smem > sm->max_smem) return 4;
    if (tmem > sm->max_tmem_cols) return 5;
    return 0;
}

int or_max_blocks(const or_smres* sm, const or_kres* k) {
    int b = 0;
    while (or_fits(sm, k, b + 1, 0, 0) == 0) ++b;
    return b;
}

/* Pruning rule read as AND with strict '<' (R9): prune iff both the PUR and the MUR
 * differences are below their thresholds. */
int or_pruned(double pur1, double mur1, double pur2, double mur2, double ap, double am) {
    return fabs(pur1 - pur2) < ap && fabs(mur1 - mur2) < am;
}
