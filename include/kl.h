/* kl.h -- C ABI of the B200-native Kernelet hot path (libkl.so).
 *
 * Kernelet (Zhong & He, arXiv:1303.5164; PAPER.md = /root/reference/PAPER.md, cited P:line)
 * runs a queue of independent GPU kernels as *slices* -- contiguous ranges of thread blocks whose
 * block index is rectified by a slice offset -- and co-schedules slices of
 * two kernels concurrently, choosing the pair and the slice ratio with a Markov-chain
 * warp-state model inside the greedy Alg.1 / FindCoSchedule.
 *
 * Conventions
 *  - Every call returns kl_status; no exception or signal crosses the ABI.  On failure a
 *    human-readable detail is kept per context (kl_last_error).  KL_ECUDA poisons the context:
 *    every later call except kl_last_error/kl_destroy returns KL_ECUDA.
 *  - All pointers inside kl_args_* structs are DEVICE pointers owned by the caller (e.g. torch
 *    tensors); they must stay valid until kl_sync returns.  The library copies descriptors, args
 *    and profiles at submit; `out` structs are caller-allocated.
 *  - Streams are cudaStream_t values passed as void*; counters_dev is a caller-owned device
 *    int64[8] buffer laid out as kl_counters (the multi-GPU layer all-gathers it over NCCL).
 *  - A context is externally synchronised (one host thread at a time); separate contexts (one
 *    per device / rank) are independent.
 *  - device = -1 creates a host-only context (no CUDA calls): submit, slice plans and profile
 *    queries work from fully specified profiles; calls that need the device (kl_predict,
 *    kl_decide on a model-cache miss, kl_schedule, kl_sync, kl_run_plain) return KL_ECUDA.
 */
#ifndef KL_H
#define KL_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KL_ABI_VERSION 3   /* 3: kl_config.distinct_kinds + reserved0 */
#define KL_MAX_SMS 256

typedef struct kl_ctx kl_ctx;

typedef enum {
    KL_OK = 0,
    KL_EINVAL = 1,       /* bad argument: Rm outside [0,1], grid_blocks = 0, unknown kind, ...   */
    KL_EINFEASIBLE = 2,  /* occupancy: detail names warps | blocks | registers | smem | TMEM     */
    KL_ENOMEM = 3,
    KL_ECUDA = 4,        /* CUDA runtime/driver error (context poisoned)                         */
    KL_ENCCL = 5,        /* reserved for the multi-GPU layer                                     */
    KL_ENUMERIC = 6,     /* reducible Markov chain: latency guard L > W_v failed or GTH pivot 0  */
    KL_EBUSY = 7,        /* a phase is in flight where none may be                                */
    KL_ENOTFOUND = 8     /* unknown kernel id / nothing pending                                  */
} kl_status;

/* The paper's eight benchmark kernels (tb:description) plus the MatrixAdd slicing
 * example and the synthetic "testing kernel". */
typedef enum {
    KL_PC = 0, KL_SAD = 1, KL_SPMV = 2, KL_ST = 3, KL_MM = 4, KL_MRIQ = 5, KL_BS = 6, KL_TEA = 7,
    KL_MATADD = 8, KL_SYNTH = 9, KL_NKINDS = 10
} kl_kind;

/* ---- kernel arguments (device pointers; layouts in DESIGN.md §4) ------------------------- */
typedef struct {   /* PC: 256 threads/block; thread t: p = (t*2654435761 mod 2^32) mod n_nodes,  */
    const int32_t* next;   /* then `hops` times p = next[p]; out[t] = p, acc[t] = sum of p (u32) */
    int32_t* out;
    uint32_t* acc;
    uint32_t n_nodes, hops, n_threads;   /* n_threads multiple of 256 */
} kl_args_pc;
typedef struct {   /* SAD: 32 threads/block, one 16x16 macroblock per block, 33x33 offsets      */
    const uint8_t* cur;    /* width x height u8, row-major */
    const uint8_t* ref;
    uint16_t* out;         /* [n_mb][33*33], index m*1089 + dy*33 + dx, displacement (dx-16,dy-16) */
    int32_t width, height; /* multiples of 16 */
} kl_args_sad;
typedef struct {   /* SPMV: CSR, one warp per row, 8 rows per block                              */
    const int32_t* rowptr; const int32_t* cols; const float* vals; const float* x;
    float* y;
    int32_t n_rows;
} kl_args_spmv;
typedef struct {   /* ST: 7-point stencil, in[z][y][x]; block = 128x4 (x,y) tile x 32 z-points, nx % 4 == 0 */
    const float* in; float* out;
    int32_t nx, ny, nz;
    float c0, c1;          /* interior out = c1*(6 neighbours) - c0*in; boundary out = in */
} kl_args_st;
typedef struct {   /* MM: C[M][N] (fp32) = A[M][K] (bf16) * B, B given K-major as Bt[N][K] (bf16);
                      one thread block = one 256x256 output tile on a CTA pair (tcgen05 2-SM)   */
    const uint16_t* A; const uint16_t* Bt;
    float* C;
    int32_t M, N, K;       /* M multiple of 256, N multiple of 256, K multiple of 64 */
} kl_args_mm;
typedef struct {   /* MRIQ: Q[i] = sum_k phiMag_k exp(i 2 pi k.x_i); one voxel per thread       */
    const float *x, *y, *z, *kx, *ky, *kz, *phimag;
    float *qr, *qi;
    int32_t num_x, num_k;
} kl_args_mriq;
typedef struct {   /* BS: European call/put (SDK BlackScholes), 2560 options per block          */
    const float *S, *X, *T;
    float *call, *put;
    int64_t n;             /* multiple of 4 */
    float R, V;
} kl_args_bs;
typedef struct {   /* TEA: 32-cycle encryption of n 64-bit blocks (v0,v1), 1280 per block       */
    const uint32_t* in; uint32_t* out;
    int64_t n;             /* multiple of 2 */
    uint32_t key[4];
} kl_args_tea;
typedef struct {   /* MATADD: C = A + B, n x n, 16x16 threads per block                         */
    const float *A, *B; float* C;
    int32_t n;             /* multiple of 16 */
} kl_args_matadd;
typedef struct {   /* SYNTH: y = f^fmas(x), f(v) = fmaf(v,a,b); 256 threads x 4 float4 per block*/
    const float* x; float* y;
    int64_t n;             /* multiple of 4 */
    int32_t fmas;
    float a, b;
} kl_args_synth;

/* ---- model inputs ------------------------------------------------------------------------ */
/* Per-kind profile (tb:para P:768-793; A24 P:1055-1060; PUR/MUR P:675-694).  Resource fields
 * left 0 are filled from the compiled kernel (cudaFuncGetAttributes / occupancy calculator). */
typedef struct {
    double rm;             /* memory instruction ratio R_m in [0,1] */
    double r;              /* memory requests per memory instruction (outstanding-request weight) */
    double ipb;            /* warp instructions per thread block, I_K of Eq.8 */
    double pur, mur;       /* pruning features */
    int32_t wpb;           /* warps per block */
    int32_t regs;          /* registers per thread */
    int32_t smem;          /* shared memory per block, bytes (static + dynamic) */
    int32_t tmem;          /* TMEM columns per block */
    int32_t bmax;          /* solo max resident blocks per SM */
    int32_t m_min;         /* p% rule: minimum slice in waves of b*n_sm blocks */
    double ipc_max;        /* pipe ceiling per virtual SM (R26; 0 = 1, the paper's model) */
    int32_t pipe;          /* id of the pipe that ceiling belongs to (0 none, 1 MUFU, 2 ALU, 3 FMA) */
    int32_t pad;
    double uc;             /* f1: fraction of memory instructions that are
                              uncoalesced (0 = all coalesced: the two-state model) */
    double ru;             /* requests per uncoalesced memory instruction (r: per coalesced one) */
} kl_profile;

typedef struct {
    double alpha_p, alpha_m;   /* pruning thresholds (defaults 0.4 / 0.1) */
    double p_percent;          /* slicing overhead limit, default 2 */
    double L0, B, a0, b0;      /* latency L(n) = L0 + a0*n/B + b0 (reading R2 of P:875) */
    double cp_min;             /* co-run only if the best predicted CP exceeds this (R25; 0 = paper) */
    int32_t n_sched;           /* warp schedulers per SM -> virtual SM; 4 on B200 */
    int32_t latency_mode;      /* 0 linear-in-requests (R2), 1 verbatim P:875 */
    int32_t level_mode;        /* 0: every b with b*wpb % n_sched == 0; 1: four levels (config C2) */
    int32_t split_rule;        /* slice ratio per pair: 0 argmin dT (Eq.8, the paper); 1 argmax CP */
    int32_t model_frozen;      /* 1: decide from installed predictions only (OPT, kl_cache_put) */
    int32_t n_sms;             /* 0 = from the device */
    int32_t chunk;             /* virtual blocks per work fetch; 0 = per-kind default */
    int32_t audit;             /* 1: count executions per virtual block (coverage audit);
                                  2: also record each block's start and end time (kl_timeline) */
    int32_t retune;            /* 1 (default): a re-plan that keeps a running kernel at another
                                  occupancy re-tunes it in place; 0: stop and relaunch */
    int32_t model_states;      /* 2 (default): two-state warp model; 3: kinds with
                                  uc > 0 use the three-state coalesced/uncoalesced chain (f1,
                                  P:1000-1019, reading R27) */
    int32_t granularity;       /* 0 (default): warps; 1: thread blocks as the modelling unit
                                  (reading R13: units of wpb/n_sched warps) */
    int32_t age_limit_us;      /* > 0: starvation guard (serving extension, f3; 0 = the paper's
                                  greedy): once the oldest pending kernel has waited longer than
                                  this, only co-schedules that include it are considered */
    int32_t mc_seed;           /* != 0: MC(s) comparator: every decision picks a
                                  uniformly random pending kind pair and maximal slice ratio
                                  (no model); the seed selects the random stream */
    int32_t speculative;       /* 1: while a cold-cache model batch runs, the oldest pending
                                  kernel starts solo (nothing else in flight) and the decision
                                  re-tunes or stops it (needs retune = 1); 0 (default): measured
                                  no gain on B200 (the batch then shares the SMs with it) */
    int32_t max_regs_per_sm, max_smem_per_sm, max_warps_per_sm, max_blocks_per_sm; /* 0 = device */
    int32_t mm_stages;         /* MM's occupancy level: TMA ring stages of its CTA
                                  pairs, one of 2 3 4 6 (32 KiB of shared memory each); 0
                                  (default): per co-schedule the deepest ring whose shared memory
                                  fits beside the partner's blocks (6 when MM runs solo) */
    int32_t critical;          /* 1: makespan extension of FindCoSchedule (beyond the paper, reading
                                  R29): while one pending kind's predicted remaining solo time
                                  (remaining blocks x I / IPC_solo) exceeds all the others' together,
                                  only co-schedules that include that kind are considered (the
                                  model's max CP among them); 0 (default): the paper's greedy */
    int32_t distinct_kinds;    /* 1: FindCoSchedule pairs two different kinds only (reading R31b:
                                  with saturation b_max, R31, two instances of one kind at (b1, b2)
                                  are that kind at b1 + b2 >= b_sat blocks per SM, which its
                                  occupancy sweep measures as no faster than solo); 0 (default):
                                  same-kind pairs are candidates */
    int32_t reserved0;         /* 0 */
    const kl_profile* profiles;   /* KL_NKINDS entries, or NULL for the built-in table */
    void* stream_a;            /* optional cudaStream_t: first stream of the launch pool       */
    void* stream_b;            /* optional cudaStream_t: second stream of the launch pool      */
    int64_t* counters_dev;     /* caller-owned device int64[8] (kl_counters), or NULL */
} kl_config;

typedef struct {
    kl_kind kind;
    uint32_t grid_blocks;      /* k thread blocks, IDs 0..k-1 */
    const void* args;          /* pointer to the kl_args_* struct of `kind` */
    uint32_t args_bytes;       /* sizeof that struct */
    const kl_profile* profile; /* NULL = table */
    uint64_t tag;              /* user tag, summed into the completion checksum */
    void* ready_event;         /* cudaEvent_t every launch of the kernel waits on (its inputs
                                  landed: the kernel's arrival), or NULL */
    const volatile uint32_t* ready_flag;   /* host-visible word (e.g. written by kl_arrival_clock
                                  through mapped memory): the kernel arrives when it becomes
                                  non-zero; NULL = no flag.  Checked after ready_event. */
} kl_kernel_desc;

typedef struct { uint32_t slice_blocks, n_slices, blocks_per_sm, waves; } kl_slice_plan;
typedef struct { int32_t k1, k2; uint32_t b1, b2; } kl_candidate;      /* kinds, blocks per SM */
typedef struct { double ipc1, ipc2, c, solo1, solo2, cp, dT; int32_t status, pad; } kl_prediction;
typedef struct {
    uint64_t id1, id2;         /* kernel ids; id2 = 0 and solo = 1 for a solo co-schedule */
    int32_t kind1, kind2;
    uint32_t b1, b2;           /* resident blocks per SM (occupancy caps) */
    uint32_t size1, size2;     /* slice sizes in blocks */
    double cp;                 /* predicted co-scheduling profit (Eq.1) */
    int32_t solo, n_candidates;
} kl_coschedule;
typedef struct {
    int64_t kernels_done, blocks_done, t_start_ns, t_end_ns, checksum, rank, world, phases;
} kl_counters;
typedef struct {               /* runtime statistics since kl_create */
    int64_t decisions;         /* FindCoSchedule decisions */
    int64_t launches;          /* persistent slice launches */
    int64_t stops;             /* stop requests (re-plans that changed a running kernel) */
    int64_t model_batches, model_candidates;
    int64_t device_launches;   /* every kernel launched by the library (incl. model, stop, init) */
    int64_t decide_ns;         /* host time spent in FindCoSchedule (incl. model batches) */
    int64_t model_ns;          /* host time spent waiting for model batches */
    int64_t retunes;           /* in-place occupancy changes of a running kernel (no stop) */
    int64_t topups;            /* top-up grids launched by re-tunes that raised the occupancy */
    int64_t aged;              /* decisions restricted by the starvation guard */
    int64_t speculative;       /* speculative solo starts that hid a model batch */
    int64_t memops;            /* control words written as stream memory operations */
} kl_stats;
typedef struct {               /* one launch of a kernel (trace / residency evidence) */
    uint64_t id;
    int32_t kind, lane;        /* lane = stream of the launch pool */
    uint32_t cap, slice, start, end, executed, admitted, max_per_sm, exhausted;
    int64_t t0_ns, t1_ns;      /* first admitted block start, last block end (globaltimer) */
    int32_t phase;             /* index of the FindCoSchedule decision that launched it */
    int32_t partner_kind;      /* kind co-scheduled by that decision, -1 = solo */
    double cp;                 /* predicted CP of that decision */
    uint32_t cap_max;          /* largest cap in force during the launch (re-tunes) */
    uint32_t grids;            /* device grids that served it (1 + top-ups) */
    uint32_t variant;          /* kind-specific instantiation (MM: TMA ring stages), 0 = none */
    uint32_t pad;
} kl_trace_rec;

/* ---- calls -------------------------------------------------------------------------------- */
int kl_abi_version(void);
kl_status kl_config_default(kl_config* cfg);
/* One context per CUDA device (multi-GPU = one scheduler per GPU). */
kl_status kl_create(int device, const kl_config* cfg, kl_ctx** out);
kl_status kl_destroy(kl_ctx* ctx);
const char* kl_last_error(const kl_ctx* ctx);

/* Alg.1 lines 2-3: add kernel K to the pending set R; returns its id (>= 1).
 * Errors: KL_EINVAL for an unknown kind, grid_blocks = 0 or >= 2^27, args_bytes != the kind's
 * kl_args size, Rm outside [0,1] in an attached profile, args the kind cannot use (ST: nx not a
 * multiple of 4; MM: M, N, K not multiples of the 256 x 256 x 64 pair tile, or grid_blocks
 * larger than the (M/256)(N/256) output tiles -- every other body range-checks its virtual block). */
kl_status kl_submit(kl_ctx* ctx, const kl_kernel_desc* desc, uint64_t* out_id);
/* kl_submit for n descriptors in order (one ABI crossing for a whole queue); out_ids[n] (may be
 * NULL).  Errors as kl_submit: the first failing descriptor's status is returned, the ones before
 * it stay submitted. */
kl_status kl_submit_batch(kl_ctx* ctx, const kl_kernel_desc* descs, size_t n, uint64_t* out_ids);
/* Slicing plan: slices of slice_blocks contiguous blocks at
 * blocks_per_sm resident blocks per SM; slice_blocks = 0 applies the p% rule (m_min waves). */
kl_status kl_slice(kl_ctx* ctx, uint64_t id, uint32_t blocks_per_sm, uint32_t slice_blocks,
                   kl_slice_plan* out);
/* Batched model on the device: one prediction per candidate.  b2 = 0 asks for the
 * solo prediction of k1 at b1 (ipc1; cp = dT = 0). */
kl_status kl_predict(kl_ctx* ctx, const kl_candidate* cands, size_t n, kl_prediction* out);
/* One step of Alg.1: wait for the next scheduling event (a kernel ran out of thread blocks, or
 * the first call), run FindCoSchedule over the pending set and reconcile the running
 * co-schedule with it (launch / stop at a slice boundary); returns without waiting for the
 * kernels.  KL_ENOTFOUND once R is empty. */
kl_status kl_schedule(kl_ctx* ctx, kl_coschedule* out);
/* Drive Alg.1 until R is empty, wait for the device, return this GPU's counters. */
kl_status kl_sync(kl_ctx* ctx, kl_counters* out);

/* Unsliced / explicitly sliced launch of one kernel: blocks [block_offset, block_offset+n_blocks)
 * run as a plain grid of n_blocks with the index rectified by block_offset.  Used by
 * the sequential and multi-stream baselines and the slicing-overhead calibration. */
kl_status kl_run_plain(kl_ctx* ctx, const kl_kernel_desc* desc, void* stream,
                       uint32_t block_offset, uint32_t n_blocks);
/* One whole kernel through the persistent slice launcher at `cap` resident blocks per SM
 * (0 = uncapped), outside the scheduler; blocks until done; *ms = device time of the launch.
 * Occupancy sweeps for the calibration (solo IPC vs warps, the E4 analog). */
kl_status kl_run_capped(kl_ctx* ctx, const kl_kernel_desc* desc, uint32_t cap, double* ms);
/* Co-run two whole kernels outside the scheduler at caps (cap1, cap2): both are launched through
 * the slice launcher, the survivor is stopped at its next fetch when the first runs out of
 * blocks, and the two launch records are returned (config C3: measured concurrent progress vs
 * the model's cIPC; E5/E7 analogs). */
kl_status kl_run_pair(kl_ctx* ctx, const kl_kernel_desc* d1, uint32_t cap1, const kl_kernel_desc* d2,
                      uint32_t cap2, kl_trace_rec out[2]);
kl_status kl_get_profile(kl_ctx* ctx, kl_kind kind, kl_profile* out);
kl_status kl_set_profile(kl_ctx* ctx, kl_kind kind, const kl_profile* p);   /* clears model cache */
kl_status kl_reset_model_cache(kl_ctx* ctx);
/* Install predictions for candidates (e.g. measured by pre-execution: the paper's OPT comparator,
 * P:1232-1233) into the prediction cache; with config.model_frozen = 1 the device model is never
 * run and a candidate without an installed prediction counts as infeasible. */
kl_status kl_cache_put(kl_ctx* ctx, const kl_candidate* cands, const kl_prediction* preds, size_t n);
kl_status kl_reset_counters(kl_ctx* ctx);  /* zero counters_dev (t_start = INT64_MAX), stream-ordered
                                              before the next launched kernel (no host sync) */
kl_status kl_trace(kl_ctx* ctx, kl_trace_rec* out, size_t cap, size_t* n_out);
/* Coverage audit (config.audit = 1): copy kernel `id`'s per-virtual-block execution counts
 * (uint32[grid_blocks], device-maintained) into host_out[0..n). */
kl_status kl_audit(kl_ctx* ctx, uint64_t id, uint32_t* host_out, size_t n);
/* Per-block start and end times (%globaltimer ns, pairs [2v, 2v+1]; 0 = never ran) of kernel
 * `id`, config.audit = 2: the measurement tools' co-run windows (progress inside the window where
 * both kernels are resident).  host_out: uint64[n], n >= 2 * grid_blocks.  Synchronises the
 * device.  Errors: KL_ENOTFOUND, KL_EINVAL (audit != 2 or n too small). */
kl_status kl_timeline(kl_ctx* ctx, uint64_t id, uint64_t* host_out, size_t n);
/* FindCoSchedule decision only (no launch) for the current pending set; runs the device model
 * on a prediction-cache miss.  KL_EBUSY while a phase is in flight. */
kl_status kl_decide(kl_ctx* ctx, kl_coschedule* out);
/* Arrival clock for online-arrival experiments (Poisson arrivals; f3): enqueue on
 * `stream` (cudaStream_t) a one-thread kernel that sleeps `ns` nanoseconds of device time after
 * it starts, then writes its release time (%globaltimer, ns) to *stamp_dev (device uint64, may
 * be NULL).  Record a kernel's ready_event on the same stream after it: the kernel arrives then.
 * Consecutive calls on one stream give cumulative arrival times.  Errors: KL_ECUDA. */
kl_status kl_delay(void* stream, uint64_t ns, uint64_t* stamp_dev);
/* Stream gate / time stamp (one thread): waits until *flag != 0 (flag may be NULL: no wait), then
 * writes %globaltimer to *stamp_dev (may be NULL).  For baselines driven by kl_arrival_clock. */
kl_status kl_wait_flag(void* stream, const volatile uint32_t* flag, uint64_t* stamp_dev);
/* Arrival clock for n arrivals in one resident thread (no per-arrival launch, so the arrivals
 * never wait for an SM slot): enqueue on `stream` a one-thread kernel that, for i = 0..n-1,
 * waits until device time t_start + gaps_dev[0] + ... + gaps_dev[i] (a cumulative schedule: a
 * late release does not delay the later ones), writes the release time (%globaltimer) to
 * stamps_dev[i] and then sets flags[i] = 1 (flags: host-mapped memory, the
 * kernels' kl_kernel_desc.ready_flag).  gaps_dev, stamps_dev: device uint64[n].  The kernel
 * occupies one warp slot of one SM until the last release.  Errors: KL_ECUDA. */
kl_status kl_arrival_clock(void* stream, const uint64_t* gaps_dev, uint64_t* stamps_dev, uint32_t* flags,
                           uint32_t n);
kl_status kl_stats_get(kl_ctx* ctx, kl_stats* out);
/* ABI self-check: writes sizeof() of kl_config, kl_profile, kl_kernel_desc, kl_slice_plan,
 * kl_candidate, kl_prediction, kl_coschedule, kl_counters, kl_trace_rec, kl_stats, then the ten
 * kl_args_* structs in kl_kind order (20 values) into out[0..n); returns how many it wrote. */
int kl_struct_sizes(uint32_t* out, int n);

#ifdef __cplusplus
}
#endif
#endif
