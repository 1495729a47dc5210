// kl_runtime.cpp -- host runtime behind include/kl.h (product path).
//
// Implements Alg.1 and Proc. FindCoSchedule over the pending set R:
//   candidate pairs -> PUR/MUR pruning (AND reading R9, halving R10/R24)
//   -> maximal occupancy splits (a5, R7) -> batched device model (kl_model.cu, cached per
//   (kind1, kind2, b1, b2)) -> selection a9 (device-fused on a cache miss, host otherwise; the
//   two are the same rules) -> reconcile the running co-schedule with the decision.
// Execution is event driven: each persistent launch (kl_launcher.cuh) raises `drained` in a
// host-mapped record when its kernel runs out of thread blocks; the host then re-plans while the
// kernel's last blocks finish, keeps the surviving kernel running when the new decision keeps its
// occupancy, stops it at a slice boundary (epoch-checked CAS, k_stop) only when the decision
// changes it, and launches successors on a pool of streams so their blocks take SM slots as the
// predecessor's tail blocks exit.
#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "kl_internal.h"

uint32_t kl_args_size(int kind);
int kl_dev_ctl_init(KlCtl* pool, const uint32_t* slots_lens, int n, unsigned long long* counters, void* stream);
int kl_mm_stage_smem(int stages);

namespace {

constexpr int kCtlPool = 16384;
constexpr int kBlob = 1024;
constexpr int kMaxCand = 8192;

// Pre-calibration defaults of the model inputs per kind (replaced by the B200 ncu calibration,
// profiles/kl_profile_b200.json, passed through kl_config.profiles).  PUR/MUR default to the
// paper's C2050 values (tb:benchmarks).
const kl_profile kDefaultProfiles[KL_NKINDS] = {
    /* PC   */ {0.25, 32.0, 720.0, 0.0096, 0.1404, 0, 0, 0, 0, 0, 1, 1.0, 0, 0},
    /* SAD  */ {0.03, 4.0, 3600.0, 0.1498, 0.1120, 0, 0, 0, 0, 0, 1, 1.0, 0, 0},
    /* SPMV */ {0.30, 8.0, 200.0, 0.3464, 0.003, 0, 0, 0, 0, 0, 1, 1.0, 0, 0},
    /* ST   */ {0.15, 4.0, 3072.0, 0.3629, 0.1156, 0, 0, 0, 0, 0, 1, 1.0, 0, 0},
    /* MM   */ {0.01, 1.0, 12000.0, 0.5804, 0.0161, 0, 0, 0, 0, 0, 1, 1.0, 0, 0},
    /* MRIQ */ {0.001, 1.0, 196608.0, 0.8539, 0.0002, 0, 0, 0, 0, 0, 1, 1.0, 0, 0},
    /* BS   */ {0.03, 16.0, 4800.0, 0.8642, 0.0604, 0, 0, 0, 0, 0, 1, 1.0, 0, 0},
    /* TEA  */ {0.01, 16.0, 15360.0, 0.9978, 0.0196, 0, 0, 0, 0, 0, 1, 1.0, 0, 0},
    /* MATADD*/ {0.30, 4.0, 80.0, 0.1, 0.1, 0, 0, 0, 0, 0, 1, 1.0, 0, 0},
    /* SYNTH*/ {0.10, 16.0, 320.0, 0.5, 0.5, 0, 0, 0, 0, 0, 1, 1.0, 0, 0},
};

constexpr int kRecRing = 1024;
constexpr int kStopRing = 256;
constexpr int kPool = 8;

struct Launch;

struct Inst {
    uint64_t id = 0, seq = 0, tag = 0;
    int kind = 0;
    uint32_t grid = 0;
    alignas(128) unsigned char blob[kBlob];
    int slot = -1;
    uint32_t next = 0;          // host view: first virtual block not yet retired
    uint32_t epoch = 0;         // launches issued (matches the control word's epoch mod 128)
    uint32_t gen = 0;           // generation of its control-block slot (membership ticket)
    bool drained = false;       // no more thread blocks (out of R)
    bool finished = false;      // drained and every launch retired
    Launch* inflight = nullptr; // at most one launch in flight per kernel
    uint32_t* audit = nullptr;
    unsigned long long* stamps = nullptr;   // audit = 2: per-block end times (timeline)
    void* ready = nullptr;      // cudaEvent_t: the kernel arrives (joins R) once it completes
    const volatile uint32_t* ready_flag = nullptr;   // host-visible arrival word (non-zero = arrived)
    int64_t t_join = 0;         // host steady-clock ns when it joined R (starvation guard)
};

inline int64_t now_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

struct Launch {
    Inst* k = nullptr;
    int rec = -1, stream = 0;
    std::vector<int> topup_streams;   // streams of top-up grids of this epoch
    uint32_t cap = 0, slice = 0, epoch = 0;
    uint32_t cap_max = 0;             // 0 = uncapped at some point
    uint32_t variant = 0;             // MM: TMA ring stages of this launch
    bool stop_requested = false;
    KlLaunch params{};
    int32_t decision = 0, partner_kind = -1;
    double cp = 0.0;
};

struct Decision {
    bool solo = true;
    int ia = 0, ib = -1;            // indices into R
    Inst* k1 = nullptr;
    Inst* k2 = nullptr;
    uint32_t b1 = 0, b2 = 0;        // caps (solo: b1 = solo level, launched uncapped)
    double cp = 0.0;
    int n_cand = 0;
};

inline double band(double x, double y) { return 1e-12 * std::max(1.0, std::max(std::fabs(x), std::fabs(y))); }

inline uint64_t cache_key(int k1, int k2, uint32_t b1, uint32_t b2) {
    return (((uint64_t)k1 * 16 + (uint64_t)k2) * 1024 + b1) * 1024 + b2;
}

// The model is symmetric in the two kernels (the joint chain of (K2,K1) is that of (K1,K2) with
// the state pair reordered): a prediction for (k2,k1,b2,b1) is the stored (k1,k2,b1,b2) one with
// the per-kernel fields swapped.
inline kl_prediction swap_pred(const kl_prediction& p) {
    kl_prediction q = p;
    q.ipc1 = p.ipc2;
    q.ipc2 = p.ipc1;
    q.solo1 = p.solo2;
    q.solo2 = p.solo1;
    return q;
}

}  // namespace

struct kl_ctx {
    int device = -1;
    bool host_only = true, poisoned = false;
    std::string err;
    kl_config cfg{};
    kl_profile prof[KL_NKINDS]{};
    KlKindInfo info[KL_NKINDS]{};
    bool info_ok[KL_NKINDS]{};
    int n_sms = 148, max_warps = 64, max_blocks = 32, max_regs = 65536, max_smem = 233472;
    cudaStream_t pool[kPool] = {};
    bool pool_own[kPool] = {};
    int pool_busy[kPool] = {};
    cudaStream_t ctrl = nullptr, stopper = nullptr;
    KlLaunchRec* recs = nullptr;       // mapped ring of launch records
    unsigned long long* stop_pinned = nullptr;   // pinned ring of stop-request words
    uint64_t stop_slot = 0;
    std::vector<int> free_recs;
    std::vector<std::unique_ptr<Launch>> inflight;
    Decision desired;
    bool have_desired = false;
    kl_stats st{};
    cudaEvent_t init_ev = nullptr;
    cudaEvent_t tune_ev = nullptr;     // re-tune write -> top-up grid ordering
    cudaEvent_t init_done[2] = {};     // last use of each init buffer
    bool init_used[2] = {};
    int init_buf = 0;
    bool reset_pending = false;        // counters reset folded into the next init launch
    KlCtl* ctl_pool = nullptr;
    std::vector<int> free_slots;
    uint32_t* init_pinned = nullptr;   // mapped (slot, len) pairs awaiting k_ctl_init (2 buffers)
    uint32_t* init_base = nullptr;
    int n_init = 0;
    bool in_schedule = false;            // decide() called by the scheduler (may launch)
    uint32_t slot_gen[kCtlPool] = {};
    std::vector<std::unique_ptr<Inst>> insts;
    std::unordered_map<uint64_t, Inst*> by_id;
    std::vector<Inst*> R;              // pending set, arrival order (Alg.1 l.1)
    int n_pending[KL_NKINDS] = {};     // instances of each kind in R (the representatives scan stops
                                       // once every pending kind has its two)
    std::vector<Inst*> arriving;       // submitted, waiting for their ready event (Alg.1 l.2)
    std::vector<std::pair<void*, bool>> ev_seen;   // per-poll cache of ready-event queries
    uint64_t next_id = 1, seq = 0;
    // model batch buffers
    double* scratch_dev = nullptr;      // general model: per-candidate chains
    int64_t scratch_cap = 0;
    int64_t* soff_pinned = nullptr;
    int64_t* soff_dev = nullptr;
    KlModelKind* mk_pinned = nullptr;
    KlModelKind* mk_dev = nullptr;
    KlCand* cand_pinned = nullptr;
    KlCand* cand_dev = nullptr;
    int32_t* off_pinned = nullptr;
    int32_t* off_dev = nullptr;
    kl_prediction* pred_dev = nullptr;
    kl_prediction* pred_pinned = nullptr;
    kl_prediction* pred_host_dev = nullptr;   // device alias of pred_pinned (mapped)
    KlCand* cand_scratch = nullptr;           // device copy of the candidates (selection)
    uint32_t* done_dev = nullptr;
    KlDecision* dec_dev = nullptr;
    KlDecision* dec_pinned = nullptr;
    std::unordered_map<uint64_t, kl_prediction> cache;
    double solo_ipc[KL_NKINDS] = {};          // IPC^solo per kind from the model's predictions
    void note_pred(const KlCand& cd, const kl_prediction& p) {
        if (p.status) return;
        if (cd.k1 >= 0 && cd.k1 < KL_NKINDS && p.solo1 > 0) solo_ipc[cd.k1] = p.solo1;
        if (cd.b2 && cd.k2 >= 0 && cd.k2 < KL_NKINDS && p.solo2 > 0) solo_ipc[cd.k2] = p.solo2;
    }
    // maximal occupancy splits per ordered kind pair (depend on the profiles only)
    std::vector<std::pair<uint32_t, uint32_t>> splits[KL_NKINDS][KL_NKINDS];
    bool splits_ok[KL_NKINDS][KL_NKINDS] = {};
    void clear_caches() {
        cache.clear();
        for (double& v : solo_ipc) v = 0.0;
        for (auto& row : splits_ok)
            for (auto& v : row) v = false;
    }
    bool lookup(int k1, int k2, uint32_t b1, uint32_t b2, kl_prediction* out) const {
        auto it = cache.find(cache_key(k1, k2, b1, b2));
        if (it != cache.end()) { if (out) *out = it->second; return true; }
        it = cache.find(cache_key(k2, k1, b2, b1));
        if (it != cache.end()) { if (out) *out = swap_pred(it->second); return true; }
        return false;
    }
    int64_t model_batches = 0, model_cands = 0;
    std::vector<kl_trace_rec> trace;
    int64_t* counters = nullptr;

    kl_status fail(kl_status st, const char* fmt, ...) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        err = buf;
        if (st == KL_ECUDA) poisoned = true;
        return st;
    }
};

#define KL_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess) return ctx->fail(KL_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)
#define KL_LIVE(ctx)                                                                         \
    do {                                                                                     \
        if (!(ctx)) return KL_EINVAL;                                                        \
        if ((ctx)->poisoned) return KL_ECUDA;                                                \
    } while (0)

namespace {

// ---- occupancy (a5) -------------------------------------------------------------
// 0 fits, else 1 warps | 2 blocks | 3 registers | 4 smem | 5 TMEM
int fits(const kl_ctx* c, const kl_profile& p1, uint32_t b1, const kl_profile* p2, uint32_t b2) {
    const kl_profile* ps[2] = {&p1, p2};
    uint32_t bs[2] = {b1, b2};
    long warps = 0, blocks = 0, regs = 0, smem = 0, tmem = 0;
    for (int i = 0; i < 2; ++i) {
        if (!ps[i] || bs[i] == 0) continue;
        long rw = ((long)ps[i]->regs * 32 + 255) / 256 * 256;
        warps += (long)bs[i] * ps[i]->wpb;
        blocks += bs[i];
        regs += (long)bs[i] * ps[i]->wpb * rw;
        smem += (long)bs[i] * (ps[i]->smem + 1024);
        tmem += (long)bs[i] * ps[i]->tmem;
    }
    if (warps > c->max_warps) return 1;
    if (blocks > c->max_blocks) return 2;
    if (regs > c->max_regs) return 3;
    if (smem > c->max_smem) return 4;
    if (tmem > 512) return 5;
    return 0;
}

// Candidate blocks-per-SM levels (a5; R14): whole warps per virtual SM.
std::vector<uint32_t> levels(const kl_ctx* c, const kl_profile& p) {
    std::vector<uint32_t> ok, out;
    const int ns = c->cfg.n_sched;
    for (int b = 1; b <= p.bmax; ++b)
        if ((b * p.wpb) % ns == 0) ok.push_back((uint32_t)b);
    if (c->cfg.level_mode == 0) return ok;
    for (int q = 1; q <= 4; ++q) {
        int t = (q * p.bmax + 3) / 4;
        for (uint32_t b : ok)
            if ((int)b >= t) {
                if (std::find(out.begin(), out.end(), b) == out.end()) out.push_back(b);
                break;
            }
    }
    return out;
}

uint32_t solo_level(const kl_ctx* c, const kl_profile& p) {
    std::vector<uint32_t> l;
    const int ns = c->cfg.n_sched;
    for (int b = p.bmax; b >= 1; --b)
        if ((b * p.wpb) % ns == 0) return (uint32_t)b;
    return 0;
}

// Maximal feasible splits (R7): feasible (b1,b2) not dominated by another feasible level pair.
std::vector<std::pair<uint32_t, uint32_t>> maximal_splits(const kl_ctx* c, const kl_profile& p1, const kl_profile& p2) {
    auto l1 = levels(c, p1), l2 = levels(c, p2);
    std::vector<std::pair<uint32_t, uint32_t>> feas, out;
    for (uint32_t a : l1)
        for (uint32_t b : l2)
            if (fits(c, p1, a, &p2, b) == 0) feas.push_back({a, b});
    for (auto& f : feas) {
        bool dom = false;
        for (auto& g : feas)
            if (g != f && g.first >= f.first && g.second >= f.second) { dom = true; break; }
        if (!dom) out.push_back(f);
    }
    std::sort(out.begin(), out.end());
    return out;
}

// MM's occupancy level (reading R28): the TMA ring depth of its CTA pairs.  The
// model sees MM at one block per SM whatever the depth (its warps do not change); the engine
// gives each launch the deepest ring whose shared memory fits beside the partner's blocks (the
// feasibility of the pair itself is decided at the shallowest ring, the kind's profile smem).
uint32_t variant_of(const kl_ctx* c, int kind, int partner_kind, uint32_t partner_b) {
    if (kind != KL_MM) return 0;
    if (c->cfg.mm_stages) return (uint32_t)c->cfg.mm_stages;
    static const int kLevels[4] = {6, 4, 3, 2};
    kl_profile pm = c->prof[KL_MM];
    const KlKindInfo& in = c->info[KL_MM];
    for (int s : kLevels) {
        pm.smem = in.static_smem + kl_mm_stage_smem(s);
        if (partner_kind < 0) {
            if (fits(c, pm, 1, nullptr, 0) == 0) return (uint32_t)s;
            continue;
        }
        const kl_profile& pp = c->prof[partner_kind];
        const uint32_t pb = partner_b ? partner_b : (uint32_t)std::max(1, pp.bmax);
        if (fits(c, pm, 1, &pp, pb) == 0) return (uint32_t)s;
    }
    return 2;
}

bool pruned(const kl_profile& a, const kl_profile& b, double ap, double am) {
    return std::fabs(a.pur - b.pur) < ap && std::fabs(a.mur - b.mur) < am;   // R9: AND, strict
}

// Eq.8 time scale of a split (the larger per-wave time I_k b_k / cIPC_k); dT ties are judged
// relative to it (R8).
double dT_scale(const kl_ctx* c, const kl_prediction& p, const KlCand& cd) {
    return std::max(c->prof[cd.k1].ipb * (double)cd.b1 / p.ipc1, c->prof[cd.k2].ipb * (double)cd.b2 / p.ipc2);
}

bool better_split(const kl_ctx* c, const kl_prediction& a, const KlCand& ca, const kl_prediction& b, const KlCand& cb,
                  int rule) {
    if (rule == 1) {   // ablation: the split with the highest predicted CP (SURVEY key finding 4)
        double t = band(a.cp, b.cp);
        if (a.cp > b.cp + t) return true;
        if (a.cp < b.cp - t) return false;
    }
    double t = 1e-9 * std::max(dT_scale(c, a, ca), dT_scale(c, b, cb));
    if (a.dT < b.dT - t) return true;
    if (a.dT > b.dT + t) return false;
    t = band(a.c, b.c);
    if (a.c > b.c + t) return true;
    if (a.c < b.c - t) return false;
    if (ca.warps != cb.warps) return ca.warps > cb.warps;
    return ca.b1 < cb.b1;
}

void fill_model_kinds(kl_ctx* c) {
    for (int k = 0; k < KL_NKINDS; ++k) {
        const kl_profile& p = c->prof[k];
        KlModelKind m{};
        m.rm = p.rm;
        m.r = p.r;
        m.ipb = p.ipb;
        m.wpb = p.wpb;
        m.bsolo = (int)solo_level(c, p);
        m.pi = (p.ipc_max > 0.0 && p.ipc_max < 1.0) ? p.ipc_max : 1.0;
        m.pipe = p.pipe;
        m.uc = p.uc;
        m.ru = p.ru > 0.0 ? p.ru : p.r;
        m.three = (c->cfg.model_states == 3 && p.uc > 0.0) ? 1 : 0;
        m.g = 1;
        if (c->cfg.granularity == 1 && p.wpb % c->cfg.n_sched == 0 && p.wpb >= c->cfg.n_sched)
            m.g = p.wpb / c->cfg.n_sched;   // a block's warps per virtual SM (R13)
        c->mk_pinned[k] = m;
    }
}

KlModelCfg model_cfg(const kl_ctx* c, int n) {
    KlModelCfg m{};
    m.L0 = c->cfg.L0;
    m.B = c->cfg.B;
    m.a0 = c->cfg.a0;
    m.b0 = c->cfg.b0;
    m.W = 64 / c->cfg.n_sched;   // virtual SM warps
    m.n_sched = c->cfg.n_sched;
    m.latency_mode = c->cfg.latency_mode;
    m.n_cand = n;
    m.split_rule = c->cfg.split_rule;
    m.preds_host = c->pred_host_dev;
    m.cands_dev = c->cand_scratch;
    return m;
}

const std::vector<std::pair<uint32_t, uint32_t>>& splits_of(kl_ctx* c, int k1, int k2) {
    if (!c->splits_ok[k1][k2]) {
        c->splits[k1][k2] = maximal_splits(c, c->prof[k1], c->prof[k2]);
        c->splits_ok[k1][k2] = true;
    }
    return c->splits[k1][k2];
}

kl_status launch_kernel(kl_ctx* ctx, Inst* k, uint32_t cap, uint32_t slice, int partner_kind, double cp,
                        uint32_t variant = 0);
uint32_t slice_of(const kl_ctx* c, uint32_t b, int m);

// The general model kernel (kl_model3.cu) serves three-state kinds and block granularity.
bool general_model(const kl_ctx* c) {
    if (c->cfg.granularity == 1) return true;
    if (c->cfg.model_states != 3) return false;
    for (int k = 0; k < KL_NKINDS; ++k)
        if (c->mk_pinned[k].three) return true;
    return false;
}

// States of one kind's chain at w warps (mirror of the device's make_kin / nstates).
int64_t kind_states(const KlModelKind& m, int w) {
    const int g = m.g > 0 ? m.g : 1;
    const int u = std::max(1, w / g);
    return m.three ? (int64_t)(u + 1) * (u + 2) / 2 : (int64_t)u + 1;
}

// Global scratch of one candidate in the general model: its largest chain's S^2 + 3 S doubles.
int64_t scratch_doubles(const kl_ctx* c, const KlCand& cd) {
    const KlModelKind& a = c->mk_pinned[cd.k1];
    const KlModelKind& b = c->mk_pinned[cd.k2];
    const int ns = c->cfg.n_sched;
    const int w1 = (int)cd.b1 * a.wpb / ns, w2 = (int)cd.b2 * b.wpb / ns;
    const int ws1 = a.bsolo * a.wpb / ns, ws2 = b.bsolo * b.wpb / ns;
    int64_t S = std::max(kind_states(a, ws1), kind_states(b, ws2));
    S = std::max(S, kind_states(a, w1) * (cd.b2 ? kind_states(b, w2) : 1));
    return S * S + 3 * S;
}

// Run the device model over cand_pinned[0..n); n_pairs > 0 fuses the selection.
kl_status run_model(kl_ctx* ctx, int n, int n_pairs, KlDecision* dec_out, Inst* spec = nullptr) {
    if (n > kMaxCand) return ctx->fail(KL_ENOMEM, "too many candidates (%d)", n);
    const auto t_model = std::chrono::steady_clock::now();
    fill_model_kinds(ctx);
    std::atomic_thread_fence(std::memory_order_seq_cst);   // mapped inputs written before the launch
    int rc;
    if (general_model(ctx)) {
        // f1 / block granularity: chains in global scratch, sized per candidate
        int64_t tot = 0;
        for (int i = 0; i < n; ++i) {
            ctx->soff_pinned[i] = tot;
            tot += scratch_doubles(ctx, ctx->cand_pinned[i]);
        }
        if (tot > ctx->scratch_cap) {
            if (ctx->scratch_dev) cudaFree(ctx->scratch_dev);
            ctx->scratch_dev = nullptr;
            ctx->scratch_cap = 0;
            KL_CUDA(cudaMalloc(&ctx->scratch_dev, sizeof(double) * (size_t)tot));
            ctx->scratch_cap = tot;
        }
        rc = kl_dev_model_general(ctx->mk_dev, model_cfg(ctx, n), ctx->cand_dev, ctx->pred_dev, n_pairs, ctx->off_dev,
                                  ctx->done_dev, ctx->dec_dev, ctx->scratch_dev, ctx->soff_dev, ctx->ctrl);
    } else {
        rc = kl_dev_model_batch(ctx->mk_dev, model_cfg(ctx, n), ctx->cand_dev, ctx->pred_dev, n_pairs, ctx->off_dev,
                                ctx->done_dev, ctx->dec_dev, ctx->ctrl);
    }
    if (rc) return ctx->fail(KL_ECUDA, "model batch launch: %s", cudaGetErrorString((cudaError_t)rc));
    if (spec && !spec->inflight && !spec->drained) {
        // speculative start: while the batch runs, the oldest pending kernel starts solo, capped
        // so that every SM keeps room for a model CTA (persistent blocks would otherwise hold the
        // SMs the model needs); the decision then re-tunes it in place or stops it
        kl_profile model_cta{};
        model_cta.wpb = 8;
        model_cta.regs = 80;
        model_cta.smem = 58 * 1024;
        const kl_profile& p0 = ctx->prof[spec->kind];
        uint32_t cap = 0;
        for (uint32_t b = 1; b <= (uint32_t)std::max(1, p0.bmax); ++b)
            if (fits(ctx, p0, b, &model_cta, 1) == 0) cap = b;
        if (cap) {
            kl_status st = launch_kernel(ctx, spec, cap, slice_of(ctx, cap, 1), -1, 0.0,
                                         variant_of(ctx, spec->kind, -1, 0) ? 2u : 0u);
            if (st) return st;
            ctx->st.speculative++;
        }
    }
    KL_CUDA(cudaStreamSynchronize(ctx->ctrl));
    ctx->model_batches++;
    ctx->model_cands += n;
    ctx->st.device_launches++;
    ctx->st.model_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t_model).count();
    for (int i = 0; i < n; ++i) {
        const KlCand& cd = ctx->cand_pinned[i];
        ctx->cache[cache_key(cd.k1, cd.k2, cd.b1, cd.b2)] = ctx->pred_pinned[i];
        ctx->note_pred(cd, ctx->pred_pinned[i]);
    }
    if (dec_out) *dec_out = *ctx->dec_pinned;
    return KL_OK;
}

// Proc. FindCoSchedule over R.
kl_status find_co_schedule(kl_ctx* ctx, Decision* d) {
    *d = Decision{};
    auto& R = ctx->R;
    if (R.empty()) return ctx->fail(KL_ENOTFOUND, "nothing pending");
    // representatives: first two instances of each kind, arrival order
    std::vector<int> reps;
    int seen_k[KL_NKINDS] = {0};
    int want = 0;                      // representatives still to find (2 per kind, or fewer pending)
    for (int k = 0; k < KL_NKINDS; ++k) want += std::min(2, ctx->n_pending[k]);
    for (int i = 0; i < (int)R.size() && want > 0; ++i)
        if (seen_k[R[i]->kind] < 2) { reps.push_back(i); seen_k[R[i]->kind]++; --want; }
    std::vector<std::pair<int, int>> pairs;
    bool seen_pair[KL_NKINDS][KL_NKINDS] = {};
    for (size_t a = 0; a < reps.size(); ++a)
        for (size_t b = a + 1; b < reps.size(); ++b) {
            int ka = R[reps[a]]->kind, kb = R[reps[b]]->kind;
            int lo = std::min(ka, kb), hi = std::max(ka, kb);
            if (seen_pair[lo][hi] || (ctx->cfg.distinct_kinds && ka == kb)) continue;
            seen_pair[lo][hi] = true;
            pairs.push_back({reps[a], reps[b]});
        }
    // starvation guard (serving extension, off by default = the paper's greedy): once the oldest
    // pending kernel has waited longer than age_limit_us, only co-schedules that include it
    if (ctx->cfg.age_limit_us > 0 && now_ns() - R[0]->t_join > (int64_t)ctx->cfg.age_limit_us * 1000) {
        std::vector<std::pair<int, int>> with0;
        for (auto& pq : pairs)
            if (pq.first == 0 || pq.second == 0) with0.push_back(pq);
        pairs.swap(with0);
        ctx->st.aged++;
    }
    // pruning with relaxation
    double ap = ctx->cfg.alpha_p, am = ctx->cfg.alpha_m;
    std::vector<std::pair<int, int>> keep;
    for (int it = 0; it < 10; ++it) {
        if (it == 9) ap = am = 0.0;
        keep.clear();
        for (auto& pq : pairs)
            if (!pruned(ctx->prof[R[pq.first]->kind], ctx->prof[R[pq.second]->kind], ap, am)) keep.push_back(pq);
        if (!keep.empty() || pairs.empty()) break;
        ap *= 0.5;
        am *= 0.5;
    }
    // candidates: maximal splits of each kept pair
    int n = 0, np = 0;
    bool missing = false;
    std::vector<std::pair<int, int>> pair_of_group;
    for (auto& pq : keep) {
        const int k1 = R[pq.first]->kind, k2 = R[pq.second]->kind;
        const auto& ms = splits_of(ctx, k1, k2);
        if (ms.empty()) continue;
        ctx->off_pinned[np] = n;
        for (auto& s : ms) {
            if (n >= kMaxCand) return ctx->fail(KL_ENOMEM, "candidate space too large");
            KlCand cd{};
            cd.k1 = k1;
            cd.k2 = k2;
            cd.b1 = s.first;
            cd.b2 = s.second;
            cd.pair = np;
            cd.warps = (int)s.first * ctx->prof[k1].wpb + (int)s.second * ctx->prof[k2].wpb;
            ctx->cand_pinned[n++] = cd;
            if (!ctx->lookup(k1, k2, s.first, s.second, nullptr)) missing = true;
        }
        pair_of_group.push_back(pq);
        ++np;
    }
    ctx->off_pinned[np] = n;
    d->n_cand = n;
    int best = -1;
    double bcp = 0.0;
    if (ctx->cfg.mc_seed) {
        // MC(s) comparator: a uniformly random pair of the pending kinds and a
        // uniformly random maximal slice ratio, no model, no pruning (counter-based splitmix64
        // stream: seed x decision number)
        std::vector<int> all;
        for (auto& pq : pairs) {
            const auto& ms = splits_of(ctx, R[pq.first]->kind, R[pq.second]->kind);
            for (size_t s = 0; s < ms.size(); ++s) all.push_back((int)((&pq - &pairs[0]) * 4096 + (int)s));
        }
        if (!all.empty()) {
            uint64_t z = (uint64_t)(uint32_t)ctx->cfg.mc_seed * 0x9E3779B97F4A7C15ull + (uint64_t)ctx->st.decisions + 1;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            z ^= z >> 31;
            const int pick = all[z % all.size()];
            const auto& pq = pairs[pick / 4096];
            const auto& sp = splits_of(ctx, R[pq.first]->kind, R[pq.second]->kind)[pick % 4096];
            d->solo = false;
            d->ia = pq.first;
            d->ib = pq.second;
            d->k1 = R[d->ia];
            d->k2 = R[d->ib];
            d->b1 = sp.first;
            d->b2 = sp.second;
            d->cp = 0.0;
            return KL_OK;
        }
    }
    if (n > 0 && missing && !ctx->cfg.model_frozen) {
        if (ctx->host_only) return ctx->fail(KL_ECUDA, "host-only context cannot run the model");
        // one batch also covers every other pair of the pending kinds (unpruned, pair = -1), so
        // the later decisions of this queue are cache hits instead of mid-queue model batches
        int ne = n;
        bool have[KL_NKINDS] = {};
        for (auto* k : R) have[k->kind] = true;
        for (int a = 0; a < KL_NKINDS; ++a)
            for (int b = a; b < KL_NKINDS; ++b) {   // one order; the other is derived (swap_pred)
                if (!have[a] || !have[b]) continue;
                for (auto& sp : splits_of(ctx, a, b)) {
                    if (ctx->lookup(a, b, sp.first, sp.second, nullptr)) continue;
                    bool in_list = false;
                    for (int i = 0; i < n && !in_list; ++i) {
                        const KlCand& c = ctx->cand_pinned[i];
                        in_list = (c.k1 == a && c.k2 == b && c.b1 == sp.first && c.b2 == sp.second) ||
                                  (c.k1 == b && c.k2 == a && c.b1 == sp.second && c.b2 == sp.first);
                    }
                    if (in_list || ne >= kMaxCand) continue;
                    KlCand cd{};
                    cd.k1 = a;
                    cd.k2 = b;
                    cd.b1 = sp.first;
                    cd.b2 = sp.second;
                    cd.pair = -1;
                    cd.warps = (int)sp.first * ctx->prof[a].wpb + (int)sp.second * ctx->prof[b].wpb;
                    ctx->cand_pinned[ne++] = cd;
                }
            }
        KlDecision dec{};
        Inst* spec = (ctx->in_schedule && ctx->cfg.speculative && ctx->cfg.retune && ctx->inflight.empty()) ? R[0]
                                                                                                        : nullptr;
        kl_status st = run_model(ctx, ne, np, &dec, spec);
        if (st) return st;
        best = dec.cand;
        bcp = dec.cp;
        if (best >= 0 && !(bcp > std::max(1e-12, ctx->cfg.cp_min))) best = -1;
    } else if (n > 0) {
        // host selection with the same rules as the fused device selection
        for (int p = 0; p < np; ++p) {
            int bi = -1;
            kl_prediction bp{};
            for (int i = ctx->off_pinned[p]; i < ctx->off_pinned[p + 1]; ++i) {
                const KlCand& cd = ctx->cand_pinned[i];
                kl_prediction a{};
                if (!ctx->lookup(cd.k1, cd.k2, cd.b1, cd.b2, &a)) a.status = KL_EINFEASIBLE;   // frozen, not installed
                if (a.status != 0) continue;
                if (bi < 0 || better_split(ctx, a, cd, bp, ctx->cand_pinned[bi], ctx->cfg.split_rule)) { bi = i; bp = a; }
            }
            if (bi < 0) continue;
            if (best < 0 || bp.cp > bcp + band(bp.cp, bcp)) { best = bi; bcp = bp.cp; }
        }
        if (best >= 0 && !(bcp > std::max(1e-12, ctx->cfg.cp_min))) best = -1;
    }
    if (ctx->cfg.critical && !ctx->cfg.mc_seed && np > 1) {
        // makespan extension (R29): the kind with the largest predicted remaining solo time,
        // if it exceeds all the others' together, is the queue's critical resource and must not
        // idle -- restrict the choice to co-schedules that include it
        double T[KL_NKINDS] = {}, tot = 0.0;
        bool known = true;
        for (Inst* k : R) {
            const kl_profile& p = ctx->prof[k->kind];
            const double ipc = ctx->solo_ipc[k->kind];
            if (!(ipc > 0)) { known = false; break; }
            const double t = (double)(k->grid - std::min(k->grid, k->next)) * p.ipb / ipc;
            T[k->kind] += t;
            tot += t;
        }
        int crit = -1;
        for (int k = 0; k < KL_NKINDS; ++k)
            if (known && T[k] > 0.5 * tot && (crit < 0 || T[k] > T[crit])) crit = k;
        if (crit >= 0) {
            int rb = -1;
            double rcp = 0.0;
            for (int p = 0; p < np; ++p) {
                const KlCand& c0 = ctx->cand_pinned[ctx->off_pinned[p]];
                if (c0.k1 != crit && c0.k2 != crit) continue;
                int bi = -1;
                kl_prediction bp{};
                for (int i = ctx->off_pinned[p]; i < ctx->off_pinned[p + 1]; ++i) {
                    const KlCand& cd = ctx->cand_pinned[i];
                    kl_prediction a{};
                    if (!ctx->lookup(cd.k1, cd.k2, cd.b1, cd.b2, &a) || a.status != 0) continue;
                    if (bi < 0 || better_split(ctx, a, cd, bp, ctx->cand_pinned[bi], ctx->cfg.split_rule)) { bi = i; bp = a; }
                }
                if (bi < 0) continue;
                if (rb < 0 || bp.cp > rcp + band(bp.cp, rcp)) { rb = bi; rcp = bp.cp; }
            }
            if (rb >= 0 && rcp > std::max(1e-12, ctx->cfg.cp_min)) { best = rb; bcp = rcp; }
        }
    }
    if (best < 0) {   // solo: oldest pending kernel at its solo maximum occupancy (R25)
        d->solo = true;
        d->ia = 0;
        d->k1 = R[0];
        d->b1 = solo_level(ctx, ctx->prof[R[0]->kind]);
        d->cp = 0.0;
        return KL_OK;
    }
    const KlCand& cd = ctx->cand_pinned[best];
    d->solo = false;
    d->ia = pair_of_group[cd.pair].first;
    d->ib = pair_of_group[cd.pair].second;
    d->k1 = R[d->ia];
    d->k2 = R[d->ib];
    d->b1 = cd.b1;
    d->b2 = cd.b2;
    d->cp = bcp;
    return KL_OK;
}

kl_status decide(kl_ctx* ctx, Decision* d) {
    auto t0 = std::chrono::steady_clock::now();
    kl_status st = find_co_schedule(ctx, d);
    ctx->st.decide_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    if (st == KL_OK) ctx->st.decisions++;
    return st;
}

uint32_t slice_of(const kl_ctx* c, uint32_t b, int m) {
    return (uint32_t)std::max(1, m) * std::max(1u, b) * (uint32_t)c->n_sms;
}

// m of the p% rule for a decision: the common number of waves per slice (a9)
int waves_of(const kl_ctx* c, const Decision& d) {
    int m = std::max(1, c->prof[d.k1->kind].m_min);
    if (d.k2) m = std::max(m, c->prof[d.k2->kind].m_min);
    return m;
}

kl_status flush_ctl_init(kl_ctx* ctx) {
    if (ctx->n_init == 0 && !ctx->reset_pending) return KL_OK;
    int rc = kl_dev_ctl_init(ctx->ctl_pool, ctx->init_pinned, ctx->n_init,
                             ctx->reset_pending ? reinterpret_cast<unsigned long long*>(ctx->counters) : nullptr,
                             ctx->stopper);
    if (rc) return ctx->fail(KL_ECUDA, "ctl init: %s", cudaGetErrorString((cudaError_t)rc));
    ctx->st.device_launches++;
    // on the stopper stream: ordered after every stop / re-tune copy aimed at the slots' previous
    // kernels; the launch streams wait for it
    KL_CUDA(cudaEventRecord(ctx->init_ev, ctx->stopper));
    for (int i = 0; i < kPool; ++i) KL_CUDA(cudaStreamWaitEvent(ctx->pool[i], ctx->init_ev, 0));
    // the kernel reads the mapped list: switch to the other buffer (waited on before reuse)
    const int b = ctx->init_buf;
    KL_CUDA(cudaEventRecord(ctx->init_done[b], ctx->stopper));
    ctx->init_used[b] = true;
    ctx->init_buf = b ^ 1;
    ctx->init_pinned = ctx->init_base + (size_t)ctx->init_buf * 3 * kCtlPool;
    if (ctx->init_used[ctx->init_buf]) KL_CUDA(cudaEventSynchronize(ctx->init_done[ctx->init_buf]));
    ctx->n_init = 0;
    ctx->reset_pending = false;
    return KL_OK;
}

int pick_stream(kl_ctx* ctx) {
    int best = 0;
    for (int i = 1; i < kPool; ++i)
        if (ctx->pool_busy[i] < ctx->pool_busy[best]) best = i;
    return best;
}

kl_status launch_kernel(kl_ctx* ctx, Inst* k, uint32_t cap, uint32_t slice, int partner_kind, double cp,
                        uint32_t variant) {
    if (ctx->free_recs.empty()) return ctx->fail(KL_ENOMEM, "launch record ring exhausted");
    const KlKindInfo& inf = ctx->info[k->kind];
    auto L = std::make_unique<Launch>();
    L->k = k;
    L->rec = ctx->free_recs.back();
    ctx->free_recs.pop_back();
    L->stream = pick_stream(ctx);
    L->cap = cap;
    L->cap_max = cap;
    L->slice = slice;
    L->epoch = k->epoch++;
    L->decision = (int32_t)ctx->st.decisions;
    L->partner_kind = partner_kind;
    L->cp = cp;
    L->variant = variant;
    KlLaunchRec* rec = ctx->recs + L->rec;
    std::memset(rec, 0, sizeof(*rec));
    KlLaunch P{};
    P.ctl = ctx->ctl_pool + k->slot;
    P.cap = cap;
    P.chunk = (uint32_t)(ctx->cfg.chunk > 0 ? ctx->cfg.chunk : inf.default_chunk);
    P.n_sms = (uint32_t)ctx->n_sms;
    P.ticket = kl_ticket(k->gen, L->epoch);
    P.rec = rec;
    P.counters = reinterpret_cast<unsigned long long*>(ctx->counters);
    P.audit = k->audit;
    P.stamps = k->stamps;
    P.tag = k->tag;
    P.variant = variant;
    // grid: cap blocks per SM plus slack, so SMs whose slots free up late (the predecessor's tail
    // blocks) still receive their share; surplus blocks fail admission and exit at once
    const uint32_t per_sm = cap ? cap : (uint32_t)std::max(1, inf.bmax);
    uint32_t grid = per_sm * (uint32_t)ctx->n_sms;
    if (cap) grid += std::max((uint32_t)ctx->n_sms, grid / 4);
    const uint32_t remaining = k->grid - k->next;
    const uint32_t need = (remaining + P.chunk - 1) / P.chunk;
    if (grid > need && !cap) grid = std::max(1u, need);
    cudaStream_t s = ctx->pool[L->stream];
    if (k->ready) KL_CUDA(cudaStreamWaitEvent(s, (cudaEvent_t)k->ready, 0));
    int rc = kl_dev_launch_persistent(k->kind, k->blob, P, grid, s);
    if (rc) return ctx->fail(KL_ECUDA, "launch kind %d: %s", k->kind, cudaGetErrorString((cudaError_t)rc));
    ctx->pool_busy[L->stream]++;
    ctx->st.launches++;
    ctx->st.device_launches++;
    L->params = P;
    k->inflight = L.get();
    ctx->inflight.push_back(std::move(L));
    return KL_OK;
}

// Control-word writes (stop / re-tune) as stream memory operations (cuStreamWriteValue64: executed
// by the GPU front end, needs neither an SM -- co-runners may fill every SM -- nor a copy engine --
// a caller's bulk H2D copy would queue it for milliseconds); copy from a pinned slot if the driver
// does not offer 64-bit stream memory operations.
typedef int (*PfnWriteValue64)(void* stream, unsigned long long addr, unsigned long long value, unsigned int flags);

PfnWriteValue64 write_value64() {
    static PfnWriteValue64 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        if (std::getenv("KL_NO_MEMOPS")) return nullptr;   // A/B switch: copy-engine writes
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PfnWriteValue64>(p);
    }
    return fn;
}

kl_status write_ctl_word(kl_ctx* ctx, volatile unsigned long long* dst, unsigned long long v) {
    if (PfnWriteValue64 fn = write_value64()) {
        const int rc = fn(ctx->stopper, (unsigned long long)(uintptr_t)dst, v, 0u);
        if (rc == 0) {
            ctx->st.memops++;
            return KL_OK;
        }
        if (std::getenv("KL_DEBUG")) std::fprintf(stderr, "cuStreamWriteValue64 failed: %d\n", rc);
    } else if (std::getenv("KL_DEBUG")) {
        std::fprintf(stderr, "cuStreamWriteValue64 entry point unavailable\n");
    }
    unsigned long long* slot = ctx->stop_pinned + (ctx->stop_slot++ % kStopRing);
    *slot = v;
    KL_CUDA(cudaMemcpyAsync((void*)dst, slot, sizeof(*slot), cudaMemcpyHostToDevice, ctx->stopper));
    return KL_OK;
}

// Re-plan that keeps a running kernel but changes its occupancy (slice ratio): the copy engine
// writes the new cap into the control block; surplus blocks leave at their next fetch, and a raise
// is served by a top-up grid joining the same epoch.  No drain, no relaunch.
kl_status retune(kl_ctx* ctx, Launch* L, uint32_t cap, int partner_kind, double cp) {
    const KlKindInfo& inf = ctx->info[L->k->kind];
    const uint32_t bmax = (uint32_t)std::max(1, inf.bmax);
    const uint32_t old_eff = L->cap ? L->cap : bmax, new_eff = cap ? cap : bmax;
    kl_status ws = write_ctl_word(ctx, &ctx->ctl_pool[L->k->slot].tune, kl_tune_req(L->epoch, cap));
    if (ws) return ws;
    ctx->st.retunes++;
    L->cap = cap;
    if (L->cap_max && (cap == 0 || cap > L->cap_max)) L->cap_max = cap;
    L->partner_kind = partner_kind;
    L->cp = cp;
    L->decision = (int32_t)ctx->st.decisions;
    if (new_eff > old_eff) {
        KL_CUDA(cudaEventRecord(ctx->tune_ev, ctx->stopper));
        const int si = pick_stream(ctx);
        cudaStream_t s = ctx->pool[si];
        KL_CUDA(cudaStreamWaitEvent(s, ctx->tune_ev, 0));
        KlLaunch P = L->params;
        P.cap = cap;
        uint32_t grid = (new_eff - old_eff) * (uint32_t)ctx->n_sms;
        grid += std::max((uint32_t)ctx->n_sms, grid / 4);
        int rc = kl_dev_launch_persistent(L->k->kind, L->k->blob, P, grid, s);
        if (rc) return ctx->fail(KL_ECUDA, "top-up kind %d: %s", L->k->kind, cudaGetErrorString((cudaError_t)rc));
        ctx->pool_busy[si]++;
        L->topup_streams.push_back(si);
        ctx->st.topups++;
        ctx->st.device_launches++;
    }
    return KL_OK;
}

// Stop request (Alg.1 re-plan): the copy engine writes an epoch-tagged request into the kernel's
// control block (no SM needed -- a stop kernel could not be scheduled while the co-runners fill
// every SM); the next block that fetches work sets the boundary.
kl_status request_stop(kl_ctx* ctx, Launch* L) {
    if (L->stop_requested) return KL_OK;
    // stop at the next fetch (at least one chunk into the epoch): persistent blocks have no
    // per-slice launch cost, so waiting for the p% slice boundary would only delay the re-plan
    const uint32_t chunk = L->params.chunk ? L->params.chunk : 1u;
    kl_status ws = write_ctl_word(ctx, &ctx->ctl_pool[L->k->slot].stop_req, kl_stop_req(L->epoch, chunk));
    if (ws) return ws;
    L->stop_requested = true;
    ctx->st.stops++;
    return KL_OK;
}

// Bring the running co-schedule in line with the desired decision: stop launches the decision
// no longer wants (or wants at another occupancy), launch wanted kernels that are idle.
kl_status reconcile(kl_ctx* ctx) {
    if (!ctx->have_desired) return KL_OK;
    const Decision& d = ctx->desired;
    const int m = waves_of(ctx, d);
    struct Want { Inst* k; uint32_t cap, slice; int partner; uint32_t variant; };
    Want w[2];
    int nw = 0;
    if (d.solo) {
        w[nw++] = {d.k1, 0u, slice_of(ctx, d.b1, m), -1, variant_of(ctx, d.k1->kind, -1, 0)};
    } else {
        w[nw++] = {d.k1, d.b1, slice_of(ctx, d.b1, m), d.k2->kind, variant_of(ctx, d.k1->kind, d.k2->kind, d.b2)};
        w[nw++] = {d.k2, d.b2, slice_of(ctx, d.b2, m), d.k1->kind, variant_of(ctx, d.k2->kind, d.k1->kind, d.b1)};
    }
    for (auto& Lp : ctx->inflight) {
        Launch* L = Lp.get();
        if (L->stop_requested || L->k->drained) continue;
        int want = -1;
        for (int i = 0; i < nw; ++i)
            if (w[i].k == L->k) want = i;
        if (want < 0 || L->variant > w[want].variant) {
            // not wanted, or its shared memory (MM's ring) does not fit beside the new partner:
            // stop at the next fetch and relaunch at the wanted level
            kl_status st = request_stop(ctx, L);
            if (st) return st;
        } else if (w[want].cap != L->cap) {
            kl_status st = ctx->cfg.retune ? retune(ctx, L, w[want].cap, w[want].partner, d.cp) : request_stop(ctx, L);
            if (st) return st;
        }
    }
    for (int i = 0; i < nw; ++i) {
        Inst* k = w[i].k;
        if (k->drained || k->inflight) continue;   // running as wanted, or stopping: relaunch later
        kl_status st = launch_kernel(ctx, k, w[i].cap, w[i].slice, w[i].partner, d.cp, w[i].variant);
        if (st) return st;
    }
    return KL_OK;
}

void mark_drained(kl_ctx* ctx, Inst* k) {
    if (k->drained) return;
    k->drained = true;
    auto& R = ctx->R;
    auto it = std::find(R.begin(), R.end(), k);
    if (it != R.end()) {
        R.erase(it);
        ctx->n_pending[k->kind]--;
    }
}

// Poll the launch records.  Returns through *replan whether R changed (a kernel drained) and
// through *progress whether anything happened at all.
kl_status poll(kl_ctx* ctx, bool* replan, bool* progress) {
    // arrivals (Alg.1 l.2-3; "the arrival of new kernels trigger the recalculation")
    // every pending arrival is checked, each distinct ready event queried once per poll (the
    // instances of a kind usually share their inputs' event); arrivals need not complete in
    // submission order (e.g. copies ordered by kernel time per byte)
    if (!ctx->arriving.empty()) {
        std::vector<std::pair<void*, bool>>& seen = ctx->ev_seen;
        seen.clear();
        for (size_t i = 0; i < ctx->arriving.size();) {
            Inst* k = ctx->arriving[i];
            if (k->ready) {
                int hit = -1;
                for (size_t s = 0; s < seen.size(); ++s)
                    if (seen[s].first == k->ready) { hit = (int)s; break; }
                bool done;
                if (hit >= 0) {
                    done = seen[hit].second;
                } else {
                    cudaError_t e = cudaEventQuery((cudaEvent_t)k->ready);
                    if (e != cudaSuccess && e != cudaErrorNotReady)
                        return ctx->fail(KL_ECUDA, "ready event of kernel %llu: %s", (unsigned long long)k->id,
                                         cudaGetErrorString(e));
                    done = (e == cudaSuccess);
                    seen.push_back({k->ready, done});
                }
                if (!done) { ++i; continue; }
            }
            if (k->ready_flag && *k->ready_flag == 0u) { ++i; continue; }
            auto pos = std::upper_bound(ctx->R.begin(), ctx->R.end(), k, [](Inst* a, Inst* b) { return a->seq < b->seq; });
            k->t_join = now_ns();
            ctx->R.insert(pos, k);
            ctx->n_pending[k->kind]++;
            ctx->arriving.erase(ctx->arriving.begin() + i);
            *replan = *progress = true;
        }
    }
    for (size_t i = 0; i < ctx->inflight.size();) {
        Launch* L = ctx->inflight[i].get();
        KlLaunchRec* r = ctx->recs + L->rec;
        if (r->drained && !L->k->drained) {
            mark_drained(ctx, L->k);
            *replan = *progress = true;
        }
        if (!r->done) {
            ++i;
            continue;
        }
        std::atomic_thread_fence(std::memory_order_acquire);
        Inst* k = L->k;
        kl_trace_rec t{};
        t.id = k->id;
        t.kind = k->kind;
        t.lane = L->stream;
        t.cap = L->cap;
        t.slice = L->slice;
        t.start = r->start;
        t.end = r->end;
        t.executed = r->executed;
        t.admitted = r->admitted;
        t.max_per_sm = r->max_per_sm;
        t.exhausted = r->exhausted;
        t.t0_ns = (int64_t)r->t0;
        t.t1_ns = (int64_t)r->t1;
        t.phase = L->decision;
        t.partner_kind = L->partner_kind;
        t.cp = L->cp;
        t.cap_max = L->cap_max;
        t.grids = 1u + (uint32_t)L->topup_streams.size();
        t.variant = L->variant;
        ctx->trace.push_back(t);
        if (std::getenv("KL_PROBE_ANATOMY") && r->t_entry)   // -DKL_PROBE_ANATOMY builds (tools/launch_anatomy.py)
            std::fprintf(stderr, "anatomy kind %d entry->t0 %.2f us  t0->t1 %.2f us  t1->done %.2f us  t_entry %llu\n",
                         k->kind, ((double)r->t0 - (double)r->t_entry) / 1e3, ((double)r->t1 - (double)r->t0) / 1e3,
                         ((double)r->t_done - (double)r->t1) / 1e3, (unsigned long long)r->t_entry);
        k->next = r->end;
        k->inflight = nullptr;
        if (r->exhausted) {
            if (!k->drained) {
                mark_drained(ctx, k);
                *replan = true;
            }
            k->finished = true;
            ctx->free_slots.push_back(k->slot);
        }
        ctx->pool_busy[L->stream]--;
        for (int s : L->topup_streams) ctx->pool_busy[s]--;
        ctx->free_recs.push_back(L->rec);
        ctx->inflight.erase(ctx->inflight.begin() + i);
        *progress = true;
    }
    return KL_OK;
}

kl_status check_streams(kl_ctx* ctx) {
    for (int i = 0; i < kPool; ++i) {
        if (!ctx->pool_busy[i]) continue;
        cudaError_t e = cudaStreamQuery(ctx->pool[i]);
        if (e != cudaSuccess && e != cudaErrorNotReady)
            return ctx->fail(KL_ECUDA, "stream %d: %s", i, cudaGetErrorString(e));
    }
    return KL_OK;
}

void fill_cs(kl_ctx* ctx, const Decision& d, kl_coschedule* out) {
    if (!out) return;
    *out = kl_coschedule{};
    const int m = waves_of(ctx, d);
    out->id1 = d.k1->id;
    out->id2 = d.k2 ? d.k2->id : 0;
    out->kind1 = d.k1->kind;
    out->kind2 = d.k2 ? d.k2->kind : -1;
    out->b1 = d.b1;
    out->b2 = d.b2;
    out->size1 = slice_of(ctx, d.b1, m);
    out->size2 = d.k2 ? slice_of(ctx, d.b2, m) : 0;
    out->cp = d.cp;
    out->solo = d.solo ? 1 : 0;
    out->n_candidates = d.n_cand;
}

// One Alg.1 decision: wait for a scheduling event (unless none was made yet), decide, reconcile.
// Returns KL_ENOTFOUND when R is empty.
kl_status schedule_step(kl_ctx* ctx, kl_coschedule* out) {
    kl_status st = flush_ctl_init(ctx);
    if (st) return st;
    bool replan = !ctx->have_desired, progress = false;
    uint64_t spins = 0;
    for (;;) {
        st = poll(ctx, &replan, &progress);
        if (st) return st;
        if (progress && !replan) {          // a stopped launch ended: relaunch it if still wanted
            st = reconcile(ctx);
            if (st) return st;
            progress = false;
        }
        if (ctx->R.empty() && ctx->arriving.empty()) {
            ctx->have_desired = false;
            return ctx->fail(KL_ENOTFOUND, "nothing pending");
        }
        if (!ctx->R.empty() && (replan || ctx->inflight.empty())) break;
        _mm_pause();
        if ((++spins & 0x3FFF) == 0) {
            st = check_streams(ctx);
            if (st) return st;
        }
    }
    Decision d;
    ctx->in_schedule = true;
    st = decide(ctx, &d);
    ctx->in_schedule = false;
    if (st) return st;
    ctx->desired = d;
    ctx->have_desired = true;
    st = reconcile(ctx);
    if (st) return st;
    fill_cs(ctx, d, out);
    return KL_OK;
}

kl_status drain_all(kl_ctx* ctx) {
    uint64_t spins = 0;
    while (!ctx->inflight.empty()) {
        bool replan = false, progress = false;
        kl_status st = poll(ctx, &replan, &progress);
        if (st) return st;
        if (progress && !ctx->R.empty()) {
            st = reconcile(ctx);
            if (st) return st;
        }
        _mm_pause();
        if ((++spins & 0x3FFF) == 0) {
            st = check_streams(ctx);
            if (st) return st;
        }
    }
    return KL_OK;
}

}  // namespace

// =============================================================================================
extern "C" {

int kl_abi_version(void) { return KL_ABI_VERSION; }

int kl_struct_sizes(uint32_t* out, int n) {
    const uint32_t s[] = {sizeof(kl_config), sizeof(kl_profile), sizeof(kl_kernel_desc), sizeof(kl_slice_plan),
                          sizeof(kl_candidate), sizeof(kl_prediction), sizeof(kl_coschedule), sizeof(kl_counters),
                          sizeof(kl_trace_rec), sizeof(kl_stats), sizeof(kl_args_pc), sizeof(kl_args_sad), sizeof(kl_args_spmv),
                          sizeof(kl_args_st), sizeof(kl_args_mm), sizeof(kl_args_mriq), sizeof(kl_args_bs),
                          sizeof(kl_args_tea), sizeof(kl_args_matadd), sizeof(kl_args_synth)};
    int m = (int)(sizeof(s) / sizeof(s[0]));
    if (n < m) m = n;
    for (int i = 0; i < m; ++i) out[i] = s[i];
    return m;
}

kl_status kl_config_default(kl_config* c) {
    if (!c) return KL_EINVAL;
    *c = kl_config{};
    c->alpha_p = 0.4;          // P:1503-1504 (C2050 defaults)
    c->alpha_m = 0.1;
    c->p_percent = 2.0;
    c->L0 = 800.0;             // cycles; calibrated on B200
    c->B = 0.26;               // 32-B sectors per cycle per virtual SM at 1.34 GHz
    c->a0 = 1.0;
    c->b0 = 0.0;
    c->n_sched = 4;            // B200: 4 SMSPs per SM -> W_v = 16
    c->retune = 1;
    c->speculative = 0;   // measured: no gain (the model batch then shares the SMs with the kernel)
    return KL_OK;
}

const char* kl_last_error(const kl_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

kl_status kl_create(int device, const kl_config* cfg_in, kl_ctx** out) {
    if (!out) return KL_EINVAL;
    *out = nullptr;
    auto ctx = std::make_unique<kl_ctx>();
    if (cfg_in) ctx->cfg = *cfg_in;
    else kl_config_default(&ctx->cfg);
    kl_config& cfg = ctx->cfg;
    if (cfg.n_sched <= 0 || 64 % cfg.n_sched) return KL_EINVAL;
    if (cfg.mm_stages && cfg.mm_stages != 2 && cfg.mm_stages != 3 && cfg.mm_stages != 4 && cfg.mm_stages != 6)
        return KL_EINVAL;
    if ((cfg.distinct_kinds != 0 && cfg.distinct_kinds != 1) || cfg.reserved0) return KL_EINVAL;
    for (int k = 0; k < KL_NKINDS; ++k) ctx->prof[k] = cfg.profiles ? cfg.profiles[k] : kDefaultProfiles[k];
    cfg.profiles = nullptr;
    ctx->device = device;
    ctx->host_only = device < 0;
    if (!ctx->host_only) {
        kl_ctx* c = ctx.get();
        {
            kl_ctx* ctx = c;   // for KL_CUDA
            KL_CUDA(cudaSetDevice(device));
            cudaDeviceProp prop;
            KL_CUDA(cudaGetDeviceProperties(&prop, device));
            ctx->n_sms = prop.multiProcessorCount;
            ctx->max_warps = prop.maxThreadsPerMultiProcessor / 32;
            ctx->max_blocks = prop.maxBlocksPerMultiProcessor;
            ctx->max_regs = prop.regsPerMultiprocessor;
            ctx->max_smem = (int)prop.sharedMemPerMultiprocessor;
            if (ctx->n_sms > KL_MAX_SMS) return KL_EINVAL;
            // eager: load every kernel and constant table now, not during scheduling
            if (int rc = kl_dev_preload()) return ctx->fail(KL_ECUDA, "preload: %s", cudaGetErrorString((cudaError_t)rc));
            if (int rc = kl_dev_model_init()) return ctx->fail(KL_ECUDA, "model init: %s", cudaGetErrorString((cudaError_t)rc));
            if (int rc = kl_dev_model3_init()) return ctx->fail(KL_ECUDA, "model3 init: %s", cudaGetErrorString((cudaError_t)rc));
            for (int k = 0; k < KL_NKINDS; ++k) {
                int rc = kl_dev_kind_info(k, &ctx->info[k]);
                ctx->info_ok[k] = (rc == 0);
                if (rc && rc != -2) {
                    cudaGetLastError();
                }
                if (ctx->info_ok[k]) {
                    kl_profile& p = ctx->prof[k];
                    const KlKindInfo& in = ctx->info[k];
                    if (!p.wpb) p.wpb = in.threads / 32;
                    if (!p.regs) p.regs = in.regs;
                    if (!p.smem) p.smem = in.static_smem + in.dyn_smem;
                    if (!p.tmem) p.tmem = in.tmem_cols;
                    if (!p.bmax) p.bmax = in.bmax;
                }
            }
            for (int i = 0; i < kPool; ++i) {
                void* s = i == 0 ? cfg.stream_a : (i == 1 ? cfg.stream_b : nullptr);
                if (s) {
                    ctx->pool[i] = (cudaStream_t)s;
                } else {
                    KL_CUDA(cudaStreamCreateWithFlags(&ctx->pool[i], cudaStreamNonBlocking));
                    ctx->pool_own[i] = true;
                }
            }
            int lo = 0, hi = 0;
            KL_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            KL_CUDA(cudaStreamCreateWithPriority(&ctx->stopper, cudaStreamNonBlocking, hi));
            KL_CUDA(cudaHostAlloc(&ctx->recs, sizeof(KlLaunchRec) * kRecRing, cudaHostAllocMapped));
            KL_CUDA(cudaHostAlloc(&ctx->stop_pinned, sizeof(unsigned long long) * kStopRing, cudaHostAllocDefault));
            std::memset(ctx->recs, 0, sizeof(KlLaunchRec) * kRecRing);
            for (int r = kRecRing - 1; r >= 0; --r) ctx->free_recs.push_back(r);
            {
                int lo = 0, hi = 0;
                KL_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
                KL_CUDA(cudaStreamCreateWithPriority(&ctx->ctrl, cudaStreamNonBlocking, hi));   // model first
            }
            KL_CUDA(cudaEventCreateWithFlags(&ctx->init_ev, cudaEventDisableTiming));
            KL_CUDA(cudaEventCreateWithFlags(&ctx->tune_ev, cudaEventDisableTiming));
            KL_CUDA(cudaMalloc(&ctx->ctl_pool, sizeof(KlCtl) * kCtlPool));
            KL_CUDA(cudaMemset(ctx->ctl_pool, 0, sizeof(KlCtl) * kCtlPool));
            KL_CUDA(cudaHostAlloc(&ctx->init_base, sizeof(uint32_t) * 6 * kCtlPool, cudaHostAllocMapped));
            ctx->init_pinned = ctx->init_base;
            for (auto& e : ctx->init_done) KL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            // model I/O in host-mapped memory: the batch reads its candidates and writes its
            // predictions over PCIe directly (no copy-engine transfer that could queue behind a
            // caller's bulk H2D copy)
            KL_CUDA(cudaHostAlloc(&ctx->mk_pinned, sizeof(KlModelKind) * KL_NKINDS, cudaHostAllocMapped));
            KL_CUDA(cudaHostGetDevicePointer((void**)&ctx->mk_dev, ctx->mk_pinned, 0));
            KL_CUDA(cudaHostAlloc(&ctx->soff_pinned, sizeof(int64_t) * kMaxCand, cudaHostAllocMapped));
            KL_CUDA(cudaHostGetDevicePointer((void**)&ctx->soff_dev, ctx->soff_pinned, 0));
            KL_CUDA(cudaHostAlloc(&ctx->cand_pinned, sizeof(KlCand) * kMaxCand, cudaHostAllocMapped));
            KL_CUDA(cudaHostGetDevicePointer((void**)&ctx->cand_dev, ctx->cand_pinned, 0));
            KL_CUDA(cudaHostAlloc(&ctx->off_pinned, sizeof(int32_t) * (kMaxCand + 1), cudaHostAllocMapped));
            KL_CUDA(cudaHostGetDevicePointer((void**)&ctx->off_dev, ctx->off_pinned, 0));
            KL_CUDA(cudaHostAlloc(&ctx->pred_pinned, sizeof(kl_prediction) * kMaxCand, cudaHostAllocMapped));
            KL_CUDA(cudaHostGetDevicePointer((void**)&ctx->pred_host_dev, ctx->pred_pinned, 0));
            KL_CUDA(cudaMalloc(&ctx->pred_dev, sizeof(kl_prediction) * (kMaxCand + KL_NKINDS)));   // + per-kind solo slots
            KL_CUDA(cudaMalloc(&ctx->cand_scratch, sizeof(KlCand) * kMaxCand));
            KL_CUDA(cudaMalloc(&ctx->done_dev, sizeof(uint32_t)));
            KL_CUDA(cudaMemset(ctx->done_dev, 0, sizeof(uint32_t)));
            KL_CUDA(cudaHostAlloc(&ctx->dec_pinned, sizeof(KlDecision), cudaHostAllocMapped));
            KL_CUDA(cudaHostGetDevicePointer((void**)&ctx->dec_dev, ctx->dec_pinned, 0));
        }
    } else {
        ctx->cand_pinned = new KlCand[kMaxCand];
        ctx->off_pinned = new int32_t[kMaxCand + 1];
    }
    if (cfg.max_regs_per_sm) ctx->max_regs = cfg.max_regs_per_sm;
    if (cfg.max_smem_per_sm) ctx->max_smem = cfg.max_smem_per_sm;
    if (cfg.max_warps_per_sm) ctx->max_warps = cfg.max_warps_per_sm;
    if (cfg.max_blocks_per_sm) ctx->max_blocks = cfg.max_blocks_per_sm;
    if (cfg.n_sms > 0) ctx->n_sms = cfg.n_sms;
    ctx->counters = cfg.counters_dev;
    for (int s = kCtlPool - 1; s >= 0; --s) ctx->free_slots.push_back(s);
    *out = ctx.release();
    return KL_OK;
}

kl_status kl_destroy(kl_ctx* ctx) {
    if (!ctx) return KL_EINVAL;
    if (!ctx->host_only) {
        if (!ctx->poisoned) cudaDeviceSynchronize();
        for (int i = 0; i < kPool; ++i)
            if (ctx->pool_own[i] && ctx->pool[i]) cudaStreamDestroy(ctx->pool[i]);
        if (ctx->stopper) cudaStreamDestroy(ctx->stopper);
        if (ctx->recs) cudaFreeHost(ctx->recs);
        if (ctx->stop_pinned) cudaFreeHost(ctx->stop_pinned);
        for (auto& k : ctx->insts) {
            if (k->audit) cudaFree(k->audit);
            if (k->stamps) cudaFree(k->stamps);
        }
        if (ctx->ctrl) cudaStreamDestroy(ctx->ctrl);
        if (ctx->init_ev) cudaEventDestroy(ctx->init_ev);
        if (ctx->tune_ev) cudaEventDestroy(ctx->tune_ev);
        cudaFree(ctx->ctl_pool);
        cudaFreeHost(ctx->init_base);
        for (auto& e : ctx->init_done) if (e) cudaEventDestroy(e);
        cudaFreeHost(ctx->mk_pinned);
        if (ctx->soff_pinned) cudaFreeHost(ctx->soff_pinned);
        if (ctx->pred_dev) cudaFree(ctx->pred_dev);
        if (ctx->cand_scratch) cudaFree(ctx->cand_scratch);
        if (ctx->scratch_dev) cudaFree(ctx->scratch_dev);
        cudaFreeHost(ctx->cand_pinned);
        cudaFreeHost(ctx->off_pinned);
        cudaFreeHost(ctx->pred_pinned);
        cudaFree(ctx->done_dev);
        cudaFreeHost(ctx->dec_pinned);
    } else {
        delete[] ctx->cand_pinned;
        delete[] ctx->off_pinned;
    }
    delete ctx;
    return KL_OK;
}

kl_status kl_submit(kl_ctx* ctx, const kl_kernel_desc* d, uint64_t* out_id) {
    KL_LIVE(ctx);
    if (!d || d->kind < 0 || d->kind >= KL_NKINDS) return ctx->fail(KL_EINVAL, "bad kind");
    if (d->grid_blocks == 0 || d->grid_blocks >= KL_MAX_GRID) return ctx->fail(KL_EINVAL, "grid_blocks out of range");
    if (!d->args || d->args_bytes != kl_args_size(d->kind))
        return ctx->fail(KL_EINVAL, "args_bytes %u != sizeof(kl_args) %u for kind %d", d->args_bytes, kl_args_size(d->kind), d->kind);
    if (d->profile) {
        const kl_profile& p = *d->profile;
        if (!(p.rm >= 0.0 && p.rm <= 1.0)) return ctx->fail(KL_EINVAL, "Rm outside [0,1]");
        ctx->prof[d->kind] = p;
        ctx->clear_caches();
    }
    if (!ctx->host_only && !ctx->info_ok[d->kind]) return ctx->fail(KL_EINVAL, "kind %d not available in this build", d->kind);
    if (ctx->free_slots.empty()) return ctx->fail(KL_ENOMEM, "slice control pool exhausted");
    auto k = std::make_unique<Inst>();
    k->id = ctx->next_id++;
    k->seq = ctx->seq++;
    k->kind = d->kind;
    k->grid = d->grid_blocks;
    k->tag = d->tag;
    k->ready = d->ready_event;
    k->ready_flag = d->ready_flag;
    if (!ctx->host_only) {
        if (kl_dev_prepare(d->kind, d->args, d->args_bytes, d->grid_blocks, k->blob, kBlob))
            return ctx->fail(KL_EINVAL, "cannot prepare args of kind %d", d->kind);
        k->slot = ctx->free_slots.back();
        ctx->free_slots.pop_back();
        k->gen = ++ctx->slot_gen[k->slot];
        ctx->init_pinned[3 * ctx->n_init] = (uint32_t)k->slot;
        ctx->init_pinned[3 * ctx->n_init + 1] = d->grid_blocks;
        ctx->init_pinned[3 * ctx->n_init + 2] = k->gen;
        ctx->n_init++;
        if (ctx->cfg.audit) {
            KL_CUDA(cudaMalloc(&k->audit, sizeof(uint32_t) * d->grid_blocks));
            KL_CUDA(cudaMemset(k->audit, 0, sizeof(uint32_t) * d->grid_blocks));
            if (ctx->cfg.audit == 2) {
                KL_CUDA(cudaMalloc(&k->stamps, 2 * sizeof(unsigned long long) * d->grid_blocks));
                KL_CUDA(cudaMemset(k->stamps, 0, 2 * sizeof(unsigned long long) * d->grid_blocks));
            }
        }
    } else {
        std::memcpy(k->blob, d->args, d->args_bytes);
    }
    Inst* raw = k.get();
    ctx->by_id[raw->id] = raw;
    if ((raw->ready || raw->ready_flag) && !ctx->host_only) ctx->arriving.push_back(raw);   // arrives later
    else {
        raw->t_join = now_ns();
        ctx->R.push_back(raw);
        ctx->n_pending[raw->kind]++;
    }
    ctx->insts.push_back(std::move(k));
    if (out_id) *out_id = raw->id;
    return KL_OK;
}

kl_status kl_submit_batch(kl_ctx* ctx, const kl_kernel_desc* d, size_t n, uint64_t* ids) {
    KL_LIVE(ctx);
    if (n && !d) return KL_EINVAL;
    for (size_t i = 0; i < n; ++i) {
        kl_status st = kl_submit(ctx, d + i, ids ? ids + i : nullptr);
        if (st) return st;
    }
    return KL_OK;
}

kl_status kl_slice(kl_ctx* ctx, uint64_t id, uint32_t b, uint32_t slice_blocks, kl_slice_plan* out) {
    KL_LIVE(ctx);
    auto it = ctx->by_id.find(id);
    if (it == ctx->by_id.end()) return ctx->fail(KL_ENOTFOUND, "unknown id %llu", (unsigned long long)id);
    if (!out || b == 0) return ctx->fail(KL_EINVAL, "blocks_per_sm must be >= 1");
    const Inst* k = it->second;
    const kl_profile& p = ctx->prof[k->kind];
    int code = fits(ctx, p, b, nullptr, 0);
    if (code) {
        static const char* names[] = {"", "warps", "blocks", "registers", "smem", "TMEM"};
        return ctx->fail(KL_EINFEASIBLE, "%u blocks/SM of kind %d exceed %s", b, k->kind, names[code]);
    }
    uint32_t s = slice_blocks ? slice_blocks : slice_of(ctx, b, std::max(1, p.m_min));
    out->slice_blocks = s;
    out->n_slices = (k->grid + s - 1) / s;
    out->blocks_per_sm = b;
    out->waves = (s + b * ctx->n_sms - 1) / (b * ctx->n_sms);
    return KL_OK;
}

kl_status kl_predict(kl_ctx* ctx, const kl_candidate* c, size_t n, kl_prediction* out) {
    KL_LIVE(ctx);
    if (ctx->host_only) return ctx->fail(KL_ECUDA, "host-only context");
    if (n > (size_t)kMaxCand || (n && (!c || !out))) return ctx->fail(KL_EINVAL, "bad candidate list");
    for (size_t i = 0; i < n; ++i) {
        if (c[i].k1 < 0 || c[i].k1 >= KL_NKINDS || c[i].k2 < 0 || c[i].k2 >= KL_NKINDS)
            return ctx->fail(KL_EINVAL, "bad kind in candidate %zu", i);
        const kl_profile &p1 = ctx->prof[c[i].k1], &p2 = ctx->prof[c[i].k2];
        if (!(p1.rm >= 0 && p1.rm <= 1 && p2.rm >= 0 && p2.rm <= 1)) return ctx->fail(KL_EINVAL, "Rm outside [0,1]");
        KlCand cd{};
        cd.k1 = c[i].k1;
        cd.k2 = c[i].k2;
        cd.b1 = c[i].b1;
        cd.b2 = c[i].b2;
        cd.pair = -1;
        ctx->cand_pinned[i] = cd;
    }
    if (n == 0) return KL_OK;
    kl_status st = run_model(ctx, (int)n, 0, nullptr);
    if (st) return st;
    std::memcpy(out, ctx->pred_pinned, sizeof(kl_prediction) * n);
    return KL_OK;
}

kl_status kl_decide(kl_ctx* ctx, kl_coschedule* out) {
    KL_LIVE(ctx);
    if (!ctx->inflight.empty()) return ctx->fail(KL_EBUSY, "launches are in flight");
    Decision d;
    kl_status st = decide(ctx, &d);
    if (st) return st;
    fill_cs(ctx, d, out);
    return KL_OK;
}

kl_status kl_schedule(kl_ctx* ctx, kl_coschedule* out) {
    KL_LIVE(ctx);
    if (ctx->host_only) return ctx->fail(KL_ECUDA, "host-only context");
    return schedule_step(ctx, out);
}

kl_status kl_sync(kl_ctx* ctx, kl_counters* out) {
    KL_LIVE(ctx);
    if (ctx->host_only) return ctx->fail(KL_ECUDA, "host-only context");
    for (;;) {
        kl_status st = schedule_step(ctx, nullptr);
        if (st == KL_ENOTFOUND) break;
        if (st) return st;
    }
    ctx->err.clear();
    kl_status st = drain_all(ctx);
    if (st) return st;
    for (int i = 0; i < kPool; ++i) KL_CUDA(cudaStreamSynchronize(ctx->pool[i]));
    KL_CUDA(cudaStreamSynchronize(ctx->stopper));
    ctx->have_desired = false;
    if (out) {
        *out = kl_counters{};
        if (ctx->counters) {
            KL_CUDA(cudaMemcpyAsync(out, ctx->counters, sizeof(kl_counters), cudaMemcpyDeviceToHost, ctx->ctrl));
            KL_CUDA(cudaStreamSynchronize(ctx->ctrl));
        }
        out->phases = ctx->st.decisions;
    }
    return KL_OK;
}

kl_status kl_delay(void* stream, uint64_t ns, uint64_t* stamp_dev) {
    int rc = kl_dev_delay((unsigned long long)ns, reinterpret_cast<unsigned long long*>(stamp_dev), stream);
    return rc ? KL_ECUDA : KL_OK;
}

kl_status kl_wait_flag(void* stream, const volatile uint32_t* flag, uint64_t* stamp_dev) {
    int rc = kl_dev_wait_flag(flag, reinterpret_cast<unsigned long long*>(stamp_dev), stream);
    return rc ? KL_ECUDA : KL_OK;
}

kl_status kl_arrival_clock(void* stream, const uint64_t* gaps_dev, uint64_t* stamps_dev, uint32_t* flags, uint32_t n) {
    if (!n) return KL_OK;
    if (!gaps_dev || !stamps_dev || !flags) return KL_EINVAL;
    int rc = kl_dev_arrival_clock(reinterpret_cast<const unsigned long long*>(gaps_dev),
                                  reinterpret_cast<unsigned long long*>(stamps_dev), flags, n, stream);
    return rc ? KL_ECUDA : KL_OK;
}

kl_status kl_stats_get(kl_ctx* ctx, kl_stats* out) {
    KL_LIVE(ctx);
    if (!out) return KL_EINVAL;
    *out = ctx->st;
    out->model_batches = ctx->model_batches;
    out->model_candidates = ctx->model_cands;
    return KL_OK;
}

kl_status kl_run_plain(kl_ctx* ctx, const kl_kernel_desc* d, void* stream, uint32_t off, uint32_t n) {
    KL_LIVE(ctx);
    if (ctx->host_only) return ctx->fail(KL_ECUDA, "host-only context");
    if (!d || d->kind < 0 || d->kind >= KL_NKINDS || !d->args || d->args_bytes != kl_args_size(d->kind))
        return ctx->fail(KL_EINVAL, "bad descriptor");
    if ((uint64_t)off + n > d->grid_blocks) return ctx->fail(KL_EINVAL, "slice beyond grid");
    alignas(128) unsigned char blob[kBlob];
    if (kl_dev_prepare(d->kind, d->args, d->args_bytes, d->grid_blocks, blob, kBlob)) return ctx->fail(KL_EINVAL, "cannot prepare args");
    int rc = kl_dev_launch_plain(d->kind, blob, off, n, stream);
    if (rc) return ctx->fail(KL_ECUDA, "plain launch: %s", cudaGetErrorString((cudaError_t)rc));
    return KL_OK;
}

kl_status kl_run_capped(kl_ctx* ctx, const kl_kernel_desc* d, uint32_t cap, double* ms) {
    KL_LIVE(ctx);
    if (ctx->host_only) return ctx->fail(KL_ECUDA, "host-only context");
    if (!ctx->inflight.empty() || !ctx->R.empty()) return ctx->fail(KL_EBUSY, "scheduler has pending work");
    uint64_t id = 0;
    kl_status st = kl_submit(ctx, d, &id);
    if (st) return st;
    Inst* k = ctx->by_id[id];
    ctx->R.clear();                       // not scheduled: launched directly below
    for (int& c : ctx->n_pending) c = 0;
    st = flush_ctl_init(ctx);
    if (st) return st;
    // the control-block init (batched per queue in the scheduler) is not part of the launch
    KL_CUDA(cudaStreamSynchronize(ctx->stopper));
    cudaEvent_t e0, e1;
    KL_CUDA(cudaEventCreate(&e0));
    KL_CUDA(cudaEventCreate(&e1));
    int si = pick_stream(ctx);
    KL_CUDA(cudaEventRecord(e0, ctx->pool[si]));
    // measurement knob (tools/launcher_overhead.py SPIN=1): a device delay queued before the
    // launch hides the host-side launch work, as inside a scheduled queue; the caller subtracts it
    if (const char* sp = std::getenv("KL_TIMING_SPIN_NS")) {
        const unsigned long long ns = std::strtoull(sp, nullptr, 10);
        const char* st_env = std::getenv("KL_TIMING_SPIN_STAMP");   // device address: release time
        unsigned long long* stamp = st_env ? reinterpret_cast<unsigned long long*>(std::strtoull(st_env, nullptr, 10)) : nullptr;
        if (ns && kl_dev_delay(ns, stamp, ctx->pool[si])) return ctx->fail(KL_ECUDA, "spin");
    }
    ctx->pool_busy[si] -= 1000;            // launch_kernel picks the least busy stream: this one
    st = launch_kernel(ctx, k, cap, k->grid, -1, 0.0, variant_of(ctx, k->kind, -1, 0));
    ctx->pool_busy[si] += 1000;
    if (st) return st;
    KL_CUDA(cudaEventRecord(e1, ctx->pool[k->inflight->stream]));
    KL_CUDA(cudaEventSynchronize(e1));
    bool rp = false, pg = false;
    while (k->inflight) {
        st = poll(ctx, &rp, &pg);
        if (st) return st;
    }
    float f = 0.f;
    KL_CUDA(cudaEventElapsedTime(&f, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (ms) *ms = f;
    return KL_OK;
}

kl_status kl_run_pair(kl_ctx* ctx, const kl_kernel_desc* d1, uint32_t cap1, const kl_kernel_desc* d2,
                      uint32_t cap2, kl_trace_rec out[2]) {
    KL_LIVE(ctx);
    if (ctx->host_only) return ctx->fail(KL_ECUDA, "host-only context");
    if (!ctx->inflight.empty() || !ctx->R.empty()) return ctx->fail(KL_EBUSY, "scheduler has pending work");
    uint64_t id1 = 0, id2 = 0;
    kl_status st = kl_submit(ctx, d1, &id1);
    if (!st) st = kl_submit(ctx, d2, &id2);
    if (st) return st;
    Inst* k1 = ctx->by_id[id1];
    Inst* k2 = ctx->by_id[id2];
    ctx->R.clear();                       // not scheduled: launched directly below
    for (int& c : ctx->n_pending) c = 0;
    st = flush_ctl_init(ctx);
    if (st) return st;
    const size_t t0 = ctx->trace.size();
    st = launch_kernel(ctx, k1, cap1, slice_of(ctx, cap1 ? cap1 : 1, 1), k2->kind, 0.0,
                       variant_of(ctx, k1->kind, k2->kind, cap2));
    if (!st) st = launch_kernel(ctx, k2, cap2, slice_of(ctx, cap2 ? cap2 : 1, 1), k1->kind, 0.0,
                                variant_of(ctx, k2->kind, k1->kind, cap1));
    if (st) return st;
    bool stopped = false;
    uint64_t spins = 0;
    while (k1->inflight || k2->inflight) {
        bool rp = false, pg = false;
        st = poll(ctx, &rp, &pg);
        if (st) return st;
        if (!stopped && (k1->drained || k2->drained)) {   // first one ran out of blocks
            Inst* other = k1->drained ? k2 : k1;
            if (other->inflight && !other->drained) {
                st = request_stop(ctx, other->inflight);
                if (st) return st;
            }
            stopped = true;
        }
        _mm_pause();
        if ((++spins & 0x3FFF) == 0) {
            st = check_streams(ctx);
            if (st) return st;
        }
    }
    if (ctx->trace.size() < t0 + 2) return ctx->fail(KL_ECUDA, "pair run lost a record");
    for (size_t i = t0; i < ctx->trace.size(); ++i) {
        const kl_trace_rec& t = ctx->trace[i];
        if (t.id == id1) out[0] = t;
        if (t.id == id2) out[1] = t;
    }
    // the stopped kernel keeps its remainder; it is not part of any queue
    for (Inst* k : {k1, k2})
        if (!k->finished) {
            k->drained = k->finished = true;
            ctx->free_slots.push_back(k->slot);
        }
    return KL_OK;
}

kl_status kl_get_profile(kl_ctx* ctx, kl_kind kind, kl_profile* out) {
    KL_LIVE(ctx);
    if (kind < 0 || kind >= KL_NKINDS || !out) return KL_EINVAL;
    *out = ctx->prof[kind];
    return KL_OK;
}

kl_status kl_set_profile(kl_ctx* ctx, kl_kind kind, const kl_profile* p) {
    KL_LIVE(ctx);
    if (kind < 0 || kind >= KL_NKINDS || !p) return KL_EINVAL;
    if (!(p->rm >= 0.0 && p->rm <= 1.0)) return ctx->fail(KL_EINVAL, "Rm outside [0,1]");
    if (!(p->uc >= 0.0 && p->uc <= 1.0)) return ctx->fail(KL_EINVAL, "uncoalesced fraction outside [0,1]");
    kl_profile q = *p;
    const kl_profile& cur = ctx->prof[kind];
    if (!q.wpb) q.wpb = cur.wpb;
    if (!q.regs) q.regs = cur.regs;
    if (!q.smem) q.smem = cur.smem;
    if (!q.tmem) q.tmem = cur.tmem;
    if (!q.bmax) q.bmax = cur.bmax;
    if (!q.m_min) q.m_min = cur.m_min;
    if (!(q.ipc_max > 0.0)) q.ipc_max = cur.ipc_max > 0.0 ? cur.ipc_max : 1.0;
    ctx->prof[kind] = q;
    ctx->clear_caches();
    return KL_OK;
}

kl_status kl_cache_put(kl_ctx* ctx, const kl_candidate* c, const kl_prediction* p, size_t n) {
    KL_LIVE(ctx);
    if (n && (!c || !p)) return KL_EINVAL;
    for (size_t i = 0; i < n; ++i) {
        if (c[i].k1 < 0 || c[i].k1 >= KL_NKINDS || c[i].k2 < 0 || c[i].k2 >= KL_NKINDS) return KL_EINVAL;
        ctx->cache[cache_key(c[i].k1, c[i].k2, c[i].b1, c[i].b2)] = p[i];
        KlCand cd{};
        cd.k1 = c[i].k1;
        cd.k2 = c[i].k2;
        cd.b1 = c[i].b1;
        cd.b2 = c[i].b2;
        ctx->note_pred(cd, p[i]);
    }
    return KL_OK;
}

kl_status kl_reset_model_cache(kl_ctx* ctx) {
    KL_LIVE(ctx);
    ctx->cache.clear();   // predictions only; the split tables depend on the profiles alone
    return KL_OK;
}

kl_status kl_reset_counters(kl_ctx* ctx) {
    KL_LIVE(ctx);
    if (ctx->host_only || !ctx->counters) return KL_OK;
    ctx->reset_pending = true;   // done by the next init launch, stream-ordered before any kernel
    return KL_OK;
}

kl_status kl_trace(kl_ctx* ctx, kl_trace_rec* out, size_t cap, size_t* n_out) {
    KL_LIVE(ctx);
    size_t n = std::min(cap, ctx->trace.size());
    if (out && n) std::memcpy(out, ctx->trace.data(), n * sizeof(kl_trace_rec));
    if (n_out) *n_out = ctx->trace.size();
    return KL_OK;
}

kl_status kl_timeline(kl_ctx* ctx, uint64_t id, uint64_t* host_out, size_t n) {
    KL_LIVE(ctx);
    auto it = ctx->by_id.find(id);
    if (it == ctx->by_id.end()) return ctx->fail(KL_ENOTFOUND, "no kernel %llu", (unsigned long long)id);
    Inst* k = it->second;
    if (!k->stamps) return ctx->fail(KL_EINVAL, "timeline disabled (config.audit != 2)");
    if (!host_out || n < 2 * (size_t)k->grid) return KL_EINVAL;
    KL_CUDA(cudaDeviceSynchronize());
    KL_CUDA(cudaMemcpy(host_out, k->stamps, 2 * sizeof(uint64_t) * k->grid, cudaMemcpyDeviceToHost));
    return KL_OK;
}

kl_status kl_audit(kl_ctx* ctx, uint64_t id, uint32_t* host_out, size_t n) {
    KL_LIVE(ctx);
    auto it = ctx->by_id.find(id);
    if (it == ctx->by_id.end()) return ctx->fail(KL_ENOTFOUND, "unknown id");
    const Inst* k = it->second;
    if (!k->audit) return ctx->fail(KL_EINVAL, "audit disabled (config.audit = 0)");
    if (!host_out || n < k->grid) return ctx->fail(KL_EINVAL, "audit buffer too small");
    for (int i = 0; i < kPool; ++i) KL_CUDA(cudaStreamSynchronize(ctx->pool[i]));
    KL_CUDA(cudaMemcpy(host_out, k->audit, sizeof(uint32_t) * k->grid, cudaMemcpyDeviceToHost));
    return KL_OK;
}

}  // extern "C"
