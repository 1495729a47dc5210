/* oracle.h -- plain, slow, obviously-correct CPU oracle for the Kernelet hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load liboracle.so.  The product path (paper_1303_5164_b200/) never
 * includes this header or links this library; the two share no code.
 *
 * Every function cites the PAPER.md passage (P:line) it follows; readings R1..R25 are those of
 * SURVEY.md §8(c), restated in DESIGN.md.  All model arithmetic is fp64.  Built with
 * -O2 -fno-fast-math -ffp-contract=off so that the C source order is the evaluation order.
 *
 * Index convention for kernels: `idx == NULL` computes every output element in order; otherwise
 * only the n_idx listed flat output indices are computed, written compactly to out[0..n_idx).
 */
#ifndef KL_ORACLE_H
#define KL_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------- O1: benchmark kernels, unsliced (tb:description) ------------- */
void or_pc(const int32_t* next, uint32_t n_nodes, uint32_t hops, uint32_t n_threads,
           const int64_t* idx, size_t n_idx, int32_t* out_p, uint32_t* out_acc);
void or_sad(const uint8_t* cur, const uint8_t* ref, int width, int height,
            const int64_t* idx, size_t n_idx, uint16_t* out);
void or_spmv(const int32_t* rowptr, const int32_t* cols, const float* vals, const float* x,
             int n_rows, const int64_t* idx, size_t n_idx, float* y, double* absrow);
void or_stencil(const float* in, int nx, int ny, int nz, float c0, float c1,
                const int64_t* idx, size_t n_idx, float* out, double* absmag);
void or_mm(const uint16_t* A_bf16, const uint16_t* Bt_bf16, int M, int N, int K,
           const int64_t* idx, size_t n_idx, float* C, double* absmag);
void or_mriq(const float* x, const float* y, const float* z, int num_x,
             const float* kx, const float* ky, const float* kz, const float* phimag, int num_k,
             const int64_t* idx, size_t n_idx, float* qr, float* qi, double* absmag);
void or_bs(const float* S, const float* X, const float* T, size_t n, double R, double V,
           const int64_t* idx, size_t n_idx, float* call, float* put, double* mag);
double or_cnd(double d);
void or_tea(const uint32_t* v, size_t n_pairs, const uint32_t key[4],
            const int64_t* idx, size_t n_idx, uint32_t* out);
void or_tea_decrypt(const uint32_t* v, size_t n_pairs, const uint32_t key[4], uint32_t* out);
void or_matadd(const float* A, const float* B, int n, float* C);
void or_synth(const float* x, size_t n, int fmas, float a, float b,
              const int64_t* idx, size_t n_idx, float* y);

/* ---------------- O2: Markov warp-state model ------------------------------------ */
typedef struct {
    double L0;          /* base memory latency, cycles */
    double B;           /* bandwidth of one virtual SM, requests/cycle (tb:para) */
    double a0, b0;      /* linear contention-model constants */
    int W;              /* warps of the (virtual) SM, W_v */
    int latency_mode;   /* 0: L(n) = L0 + a0*n/B + b0 (R2); 1: verbatim L0 + B/(a0*max(I,1)) + b0 */
    int pir_mode;       /* 0: P_ir = min(1, R/L) (R1); 1: P_ir = const_q (test mode, textbook pin) */
    double const_q;
} or_smcfg;

typedef struct {        /* per-kernel model descriptor (tb:para; A24 P:1055-1060) */
    double rm;          /* memory instruction ratio R_m */
    double r;           /* memory requests per memory instruction (outstanding-request weight) */
    double ipb;         /* warp instructions per thread block, I_K (Eq.8) */
    int wpb;            /* warps per block */
    double pi;          /* pipe ceiling (R26): instructions/cycle the kernel's busiest pipe allows;
                           1 (or 0) = issue-limited only, the paper's model */
    int pipe;           /* id of that pipe (0 = none); kernels with the same id share it */
} or_kmodel;

double or_latency(const or_smcfg* c, double n_outstanding, int idle_warps);
/* One kernel's idle-count transition row T(i -> j), j = 0..w, for per-warp probabilities
 * p_ir (idle->ready) and rm (ready->idle): Eq.2 constraints summed with independent-warp
 * binomial weights (R3). */
void or_row(int w, int i, double p_ir, double rm, double* row /* w+1 */);
/* Homogeneous chain over S_0..S_w.  P is (w+1)x(w+1) row-major; R[i] = round
 * duration max(w-i, 1).  Returns 0, or -1 if the L>W guard fails (R22). */
int or_build_homog(const or_kmodel* k, int w, const or_smcfg* c, double* P, double* R);
/* Joint chain over (p,q), index p*(w2+1)+q. */
int or_build_joint(const or_kmodel* k1, int w1, const or_kmodel* k2, int w2,
                   const or_smcfg* c, double* P, double* R);
/* Stationary pi: (P^T - I) pi = 0 with the last equation replaced by sum(pi) = 1, dense LU with
 * partial pivoting (Eq.3).  Returns 0, or -1 if singular. */
int or_stationary(int S, const double* P, double* pi);
double or_ipc_homog(int w, const double* pi);                                   /* Eq.4 */
double or_ipc_homog_r(int w, const double* pi, const double* R);                  /* Eq.4, R26 */
void or_ipc_joint(int w1, int w2, const double* pi, const double* R,
                  double* ipc1, double* ipc2, double* c);                         /* Eq.5-7 */
double or_cp(int n, const double* cipc, const double* ipc);                       /* Eq.1 */

typedef struct { double ipc1, ipc2, c, solo1, solo2, cp, dT; int status; } or_pred;
/* Full prediction of one candidate (k1 at b1 blocks/SM, k2 at b2) against the solo IPCs at
 * b1max / b2max (R14: w = b*wpb/nsched).  status 0 ok, 2 infeasible warps, 6 numeric. */
void or_predict(const or_kmodel* k1, int b1, int b1max, const or_kmodel* k2, int b2, int b2max,
                int nsched, const or_smcfg* c, or_pred* out);
double or_solo_ipc(const or_kmodel* k, int b, int nsched, const or_smcfg* c, int* status);

/* ---------------- O3: occupancy and pruning ---------------------------- */
/* ---------------- f1: three-state (coalesced / uncoalesced) model, P:1000-1019 (model3.c) ------ */
typedef struct {
    double rm;          /* memory instruction ratio */
    double r;           /* requests per coalesced memory instruction */
    double uc;          /* fraction of memory instructions that are uncoalesced */
    double ru;          /* requests per uncoalesced memory instruction */
    double ipb;         /* warp instructions per block (Eq.8) */
    int wpb;            /* warps per block */
    double pi;          /* pipe ceiling (R26) */
    int pipe;
    int g;              /* warps per modelling unit (R13 block granularity); 0/1 = warps */
} or_kmodel3;
int or3_nstates(int w);
void or3_row(const or_kmodel3* k, int w, int c, int u, double pc, double pu, double* row);
int or3_build(const or_kmodel3* k1, int w1, const or_kmodel3* k2, int w2, const or_smcfg* cfg, double* P,
              double* R);
void or3_ipc(int w1, int w2, int joint, const double* pi, const double* R, double* ipc1, double* ipc2);
void or3_ipc_g(int w1, int g1, int w2, int g2, int joint, const double* pi, const double* R, double* ipc1,
               double* ipc2);
double or3_solo_ipc(const or_kmodel3* k, int b, int nsched, const or_smcfg* cfg, int* status);
void or3_predict(const or_kmodel3* k1, int b1, int b1max, const or_kmodel3* k2, int b2, int b2max, int nsched,
                 const or_smcfg* cfg, or_pred* out);

typedef struct { int max_warps, max_blocks, max_regs, max_smem, max_tmem_cols, reg_unit; } or_smres;
typedef struct { int wpb, regs, smem, tmem; } or_kres;
/* Resident blocks of k1 (b1) and k2 (b2) fit one SM?  Returns 0 or a code naming the binding
 * constraint: 1 warps, 2 blocks, 3 registers, 4 shared memory, 5 TMEM. */
int or_fits(const or_smres* sm, const or_kres* k1, int b1, const or_kres* k2, int b2);
int or_max_blocks(const or_smres* sm, const or_kres* k);
/* Is the pair pruned: |dPUR| < ap AND |dMUR| < am (R9, strict). */
int or_pruned(double pur1, double mur1, double pur2, double mur2, double ap, double am);

#ifdef __cplusplus
}
#endif
#endif
