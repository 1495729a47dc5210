// kl_internal.h -- device/host shared structures of libkl (product path; not used by oracle/).
#pragma once
#include <cstdint>
#include "../../include/kl.h"

// ---------------------------------------------------------------------------------------------
// Slice control block (one per submitted kernel instance, device memory).
// A kernel's virtual block range [0, len) is consumed by work-pulling persistent blocks; the
// 64-bit `word` linearises every fetch and every stop of the current launch:
//   bits [0,28)  next    : next virtual block to hand out (absolute)
//   bits [28,56) stop_at : absolute slice boundary at which the current launch stops
//   bits [56,63) epoch   : launch counter of this kernel (mod 128)
//   bit  63      stop    : stop requested for the current launch
// Fetch = atomicAdd(word, chunk); stop = CAS (only for the expected epoch) setting stop_at to the
// first slice boundary at or after `next` (at least one slice into the launch).  Hence every
// handed-out block below the final limit runs exactly once and [limit, len) stays pending
// (every thread block in exactly one co-schedule).  len < 2^27.
// ---------------------------------------------------------------------------------------------
#define KL_W_NEXT_BITS 28
#define KL_W_MASK28 ((1ull << 28) - 1ull)
#define KL_W_STOP (1ull << 63)
#define KL_MAX_GRID (1u << 27)
#if defined(__CUDACC__)
#define KL_HD __host__ __device__ __forceinline__
#else
#define KL_HD inline
#endif
KL_HD uint32_t kl_w_next(unsigned long long w) { return (uint32_t)(w & KL_W_MASK28); }
KL_HD uint32_t kl_w_stop_at(unsigned long long w) { return (uint32_t)((w >> 28) & KL_W_MASK28); }
KL_HD uint32_t kl_w_epoch(unsigned long long w) { return (uint32_t)((w >> 56) & 0x7full); }
KL_HD unsigned long long kl_w_make(uint32_t next, uint32_t stop_at, uint32_t epoch, bool stop) {
    return ((unsigned long long)next & KL_W_MASK28) | (((unsigned long long)stop_at & KL_W_MASK28) << 28) |
           (((unsigned long long)epoch & 0x7full) << 56) | (stop ? KL_W_STOP : 0ull);
}

// Membership word of the current epoch (one epoch = one host-level launch, possibly served by
// several device grids: the first grid plus top-ups when a re-plan raises the occupancy):
//   bits [0,32) live blocks, bits [32,63) ticket, bit 63 closed.
// ticket = (slot generation << 7) | (epoch mod 128), so blocks of a finished kernel whose slot
// was recycled, or of an older epoch, never match.  A block joins with one atomicAdd (after a
// plain read filters late blocks); the block whose leave brings the count to zero closes the
// epoch -- but only once its range is finished (exhausted or stopped) -- and finalizes it from
// the control block's own record (KlCtl::fin), so even a late block undoing a stray join can.
#define KL_J_CLOSED (1ull << 63)
KL_HD uint32_t kl_ticket(uint32_t gen, uint32_t epoch) { return ((gen & 0xffffffu) << 7) | (epoch & 0x7fu); }
KL_HD unsigned long long kl_j_make(uint32_t ticket, bool closed) {
    return ((unsigned long long)(ticket & 0x7fffffffu) << 32) | (closed ? KL_J_CLOSED : 0ull);
}
KL_HD uint32_t kl_j_count(unsigned long long j) { return (uint32_t)(j & 0xffffffffull); }
KL_HD uint32_t kl_j_ticket(unsigned long long j) { return (uint32_t)((j >> 32) & 0x7fffffffull); }
KL_HD bool kl_j_closed(unsigned long long j) { return (j & KL_J_CLOSED) != 0ull; }

struct KlLaunchRec;
struct KlFin {             // what the finalizing block needs, written by every joined block
    KlLaunchRec* rec;
    unsigned long long* counters;
    unsigned long long tag;
    uint32_t n_sms, pad;
};

struct KlCtl {
    unsigned long long word;
    unsigned long long join;   // membership word (kl_j_*)
    KlFin fin;
    uint32_t len;
    uint32_t drained;     // 1 once a block found the range exhausted (kernel has no more blocks)
    uint32_t admitted;    // admitted blocks of the current launch
    uint32_t executed;    // virtual blocks executed in the current launch
    uint32_t base;        // first virtual block of the current launch (slice boundaries)
    unsigned long long t0;  // earliest admitted-block start (globaltimer ns), current launch
    // host stop request, written by the copy engine (no SM needed): bit 0 valid, bits [1,8) epoch
    // of the launch to stop, bits [32,64) slice size; the next fetching block performs the stop
    volatile unsigned long long stop_req;
    // host occupancy re-tune, written by the copy engine: bit 0 valid, bits [1,8) epoch, bits
    // [32,64) blocks per SM (0 = uncapped).  Blocks above the cap on their SM leave at their next
    // fetch; raising the cap is served by a top-up grid of the same epoch.
    volatile unsigned long long tune;
    uint32_t sm_count[KL_MAX_SMS];   // resident admitted blocks per SM (occupancy cap)
    uint32_t sm_hwm[KL_MAX_SMS];     // high-water mark per SM (residency evidence)
    // per-SM epoch statistics (no hot address at block start / exit; summed at finalize)
    uint32_t sm_adm[KL_MAX_SMS];             // admissions
    uint32_t sm_exec[KL_MAX_SMS];            // virtual blocks executed
    unsigned long long sm_t0[KL_MAX_SMS];    // earliest admitted start (0 = none)
};

// Host-mapped (pinned) record of one launch: `drained` is raised by the first block that finds
// the kernel's range exhausted, the rest by the launch's last block.
struct KlLaunchRec {
    volatile uint32_t drained;
    volatile uint32_t done;
    uint32_t start;       // first virtual block of the launch
    uint32_t end;         // first virtual block not executed (absolute)
    uint32_t exhausted;   // end == len
    uint32_t executed, admitted, max_per_sm;
    unsigned long long t0, t1;
    unsigned long long t_entry, t_done;   // -DKL_PROBE_ANATOMY builds: block 0's entry, end of finalize
};

struct KlLaunch {
    KlCtl* ctl;
    uint32_t cap;                   // admitted blocks per SM (0 = no cap)
    uint32_t chunk;                 // virtual blocks per fetch
    uint32_t n_sms;
    uint32_t ticket;                // kl_ticket(slot generation, epoch) this grid serves
    KlLaunchRec* rec;
    unsigned long long* counters;   // kl_counters on the device (may be null)
    uint32_t* audit;                // per-virtual-block execution counts (may be null)
    unsigned long long* stamps;     // per-virtual-block end time, %globaltimer (may be null)
    unsigned long long tag;
    uint32_t variant;               // kind-specific instantiation (MM: TMA ring stages; 0 = default)
    uint32_t pad;
};

// ---- kernel-side entry points exported by kl_kernels.cu / kl_mm.cu ---------------------------
struct KlKindInfo {
    int threads;          // threads per block
    int dyn_smem;         // dynamic shared memory per block
    int regs;             // registers per thread (persistent variant)
    int static_smem;
    int tmem_cols;
    int bmax;             // occupancy calculator, solo
    int default_chunk;
};

// Query attributes of the persistent variant of `kind` (needs a CUDA device).
int kl_dev_kind_info(int kind, KlKindInfo* out);
// Prepare per-instance device state (e.g. TMA descriptors for MM); `blob` receives up to
// 512 bytes of launch-time parameter data stored with the instance.
// Validate and pack a kernel's args into its launch blob.  `grid` is the descriptor's grid_blocks:
// kinds whose body indexes by the virtual block without a range guard (MM: one output tile per
// block) reject a grid larger than their arguments imply.
int kl_dev_prepare(int kind, const void* args, uint32_t args_bytes, uint32_t grid, void* blob, uint32_t blob_cap);
// Launch the persistent slice launcher for `kind` with `grid` blocks.
int kl_dev_launch_persistent(int kind, const void* blob, const KlLaunch& L, uint32_t grid,
                             void* stream);
// Launch a plain grid of n_blocks with blockIdx rectified by offset.
int kl_dev_launch_plain(int kind, const void* blob, uint32_t offset, uint32_t n_blocks,
                        void* stream);

// ---- model kernels (kl_model.cu) ---------------------------------------------------------
struct KlModelKind {       // per-kind model inputs, device table
    double rm, r, ipb, pi;    // pi: pipe ceiling (R26), 1 = none
    double uc, ru;            // f1: uncoalesced fraction of memory instructions, its requests
    int32_t wpb, bsolo, pipe;
    int32_t g;                // warps per modelling unit (R13 block granularity; 1 = warps)
    int32_t three;            // 1: three-state chain for this kind (f1)
    int32_t pad1;
};
struct KlCand;
struct KlModelCfg {
    double L0, B, a0, b0;
    int32_t W, n_sched, latency_mode, n_cand;
    int32_t split_rule, pad;
    kl_prediction* preds_host;   // host-mapped copy of the predictions (may be null)
    KlCand* cands_dev;           // device copy of the candidates (the fused selection reads it)
};
struct KlCand {            // one candidate, and its grouping for the fused selection
    int32_t k1, k2;
    uint32_t b1, b2;
    int32_t pair;          // pair index (selection groups; -1: prediction only)
    int32_t warps;         // b1*wpb1 + b2*wpb2 (tie-break)
};
struct KlDecision {
    int32_t cand;          // chosen candidate index, -1 = none (solo)
    int32_t n_pairs;
    double cp;
    volatile int32_t done;
    int32_t pad;
};
// Initialise slice control blocks from a (host-mapped) list of (slot, len, generation) triples.
int kl_dev_ctl_init(KlCtl* pool, const uint32_t* slots_lens, int n, unsigned long long* counters, void* stream);
// Stop request encoding (see KlCtl::stop_req).
KL_HD unsigned long long kl_stop_req(uint32_t epoch, uint32_t slice) {
    return 1ull | ((unsigned long long)(epoch & 0x7fu) << 1) | ((unsigned long long)slice << 32);
}

// Eager one-time setup (kl_create): load every library kernel, model constant tables.
int kl_dev_preload();
int kl_dev_model_init();
int kl_dev_model3_init();

// Arrival clock: sleep ns on `stream`, then write the release time (globaltimer) to *stamp.
int kl_dev_delay(unsigned long long ns, unsigned long long* stamp, void* stream);
int kl_dev_wait_flag(const volatile uint32_t* flag, unsigned long long* stamp, void* stream);
int kl_dev_arrival_clock(const unsigned long long* gaps, unsigned long long* stamps, uint32_t* flags, uint32_t n,
                         void* stream);

// Occupancy re-tune encoding (see KlCtl::tune).
KL_HD unsigned long long kl_tune_req(uint32_t epoch, uint32_t cap) {
    return 1ull | ((unsigned long long)(epoch & 0x7fu) << 1) | ((unsigned long long)cap << 32);
}

// General model (f1 three-state kinds and/or block-granularity units): one CTA per candidate,
// the chains in global scratch (`scratch` + `scratch_off[c]` doubles for candidate c, room for
// (S^2 + 3 S) doubles with S its largest chain); same predictions / fused selection contract.
int kl_dev_model_general(const KlModelKind* kinds, KlModelCfg cfg, const KlCand* cands,
                         kl_prediction* preds, int n_pairs, const int32_t* pair_off,
                         uint32_t* done_counter, KlDecision* dec, double* scratch,
                         const int64_t* scratch_off, void* stream);

// Batched model: one CTA per candidate plus one per kind (solo chains); `preds` holds n_cand +
// KL_NKINDS entries (the tail is scratch).  If n_pairs > 0 the last CTA to finish runs the greedy
// selection (a9) and writes *dec.  `done_counter` must be zero on entry (reset by the kernel).
int kl_dev_model_batch(const KlModelKind* kinds, KlModelCfg cfg, const KlCand* cands,
                       kl_prediction* preds, int n_pairs, const int32_t* pair_rank,
                       uint32_t* done_counter, KlDecision* dec, void* stream);
