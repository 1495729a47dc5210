// kl_launcher.cuh -- the persistent slice launcher shared by every kernel body (product path).
//
// Slicing: a slice is a contiguous range of a kernel's thread blocks launched with
// its block index rectified by an offset.  On B200 a co-schedule launches ONE persistent grid per
// kernel (cap x n_SM blocks, plus slack); each admitted block pulls virtual block ids from the
// kernel's slice control word (KlCtl::word) and runs Body::block(vb) -- index rectification as a
// kernel parameter instead of Fermi SASS rewriting.  Occupancy control is a per-SM
// admission cap read from %smid; a host re-tune (KlCtl::tune) lowers it in place (surplus blocks
// leave at their next fetch) or raises it (a top-up grid joins the same epoch), so a re-plan that
// only changes a running kernel's slice ratio costs no drain and no relaunch.  The first block to
// find the range exhausted raises the kernel's `drained` event in host-mapped memory (Alg.1 l.9:
// "K1 and K2 both still have thread blocks" turns false), which is what the host scheduler reacts
// to; a host-requested stop (KlCtl::stop_req) ends the epoch at the next fetch boundary.
// Header-only: included by kl_kernels.cu and kl_mm.cu.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <algorithm>
#include <type_traits>
#include "kl_internal.h"

namespace {

__device__ __forceinline__ uint32_t smid_u32() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t smem_u32_of(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Stop the launch of epoch `epoch` at the first slice boundary at or after `next`, at least one
// slice past its first block; no-op if already stopped or the word belongs to another launch.
__device__ void stop_word(KlCtl* ctl, uint32_t epoch, uint32_t slice) {
    unsigned long long old = atomicAdd(&ctl->word, 0ull);
    const uint32_t sl = slice ? slice : 1u;
    for (;;) {
        if ((old & KL_W_STOP) || kl_w_epoch(old) != (epoch & 0x7fu)) return;
        const uint32_t nx = kl_w_next(old), base = ctl->base;
        unsigned long long n_sl = nx > base ? ((unsigned long long)(nx - base) + sl - 1) / sl : 0ull;
        if (n_sl == 0) n_sl = 1;
        unsigned long long sa = (unsigned long long)base + n_sl * sl;
        if (sa > KL_W_MASK28) sa = KL_W_MASK28;
        const unsigned long long nw = kl_w_make(nx, (uint32_t)sa, kl_w_epoch(old), true);
        const unsigned long long prev = atomicCAS(&ctl->word, old, nw);
        if (prev == old) return;
        old = prev;
    }
}

// Effective limit of the current launch from a word value: min(len, stop_at if stopped).
__device__ __forceinline__ uint32_t word_limit(unsigned long long w, uint32_t len) {
    uint32_t lim = len;
    if (w & KL_W_STOP) lim = min(lim, kl_w_stop_at(w));
    return lim;
}

struct EpochStats {
    uint32_t mx, executed, admitted;
    unsigned long long t0;
};

// Per-SM epoch statistics gathered and reset by one thread (rare path: a late block's undo closes
// the epoch).  Every member has left, so plain L2 accesses suffice.
__device__ EpochStats gather_stats_serial(KlCtl* ctl, uint32_t n_sms) {
    EpochStats s{0u, 0u, 0u, ~0ull};
    for (uint32_t i = 0; i < n_sms && i < KL_MAX_SMS; ++i) {
        s.mx = max(s.mx, __ldcg(&ctl->sm_hwm[i]));
        s.executed += __ldcg(&ctl->sm_exec[i]);
        s.admitted += __ldcg(&ctl->sm_adm[i]);
        const unsigned long long ts = __ldcg(&ctl->sm_t0[i]);
        if (ts) s.t0 = min(s.t0, ts);
        __stcg(&ctl->sm_hwm[i], 0u);
        __stcg(&ctl->sm_exec[i], 0u);
        __stcg(&ctl->sm_adm[i], 0u);
        __stcg(&ctl->sm_t0[i], 0ull);
    }
    __threadfence();
    return s;
}

// The same by the whole closing block (normal path): one SM entry per thread, block reduction;
// the result is valid in thread 0.
template <int kThreads>
__device__ EpochStats gather_stats_block(KlCtl* ctl, uint32_t n_sms) {
    __shared__ uint32_t r_mx[kThreads / 32], r_ex[kThreads / 32], r_ad[kThreads / 32];
    __shared__ unsigned long long r_t0[kThreads / 32];
    uint32_t mx = 0, ex = 0, ad = 0;
    unsigned long long t0 = ~0ull;
    for (uint32_t i = threadIdx.x; i < n_sms && i < KL_MAX_SMS; i += kThreads) {
        mx = max(mx, __ldcg(&ctl->sm_hwm[i]));
        ex += __ldcg(&ctl->sm_exec[i]);
        ad += __ldcg(&ctl->sm_adm[i]);
        const unsigned long long ts = __ldcg(&ctl->sm_t0[i]);
        if (ts) t0 = min(t0, ts);
        __stcg(&ctl->sm_hwm[i], 0u);
        __stcg(&ctl->sm_exec[i], 0u);
        __stcg(&ctl->sm_adm[i], 0u);
        __stcg(&ctl->sm_t0[i], 0ull);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        ex += __shfl_xor_sync(0xffffffffu, ex, o);
        ad += __shfl_xor_sync(0xffffffffu, ad, o);
        t0 = min(t0, __shfl_xor_sync(0xffffffffu, t0, o));
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { r_mx[w] = mx; r_ex[w] = ex; r_ad[w] = ad; r_t0[w] = t0; }
    __threadfence();
    __syncthreads();
    EpochStats s{0u, 0u, 0u, ~0ull};
    if (threadIdx.x == 0)
        for (int i = 0; i < kThreads / 32; ++i) {
            s.mx = max(s.mx, r_mx[i]);
            s.executed += r_ex[i];
            s.admitted += r_ad[i];
            s.t0 = min(s.t0, r_t0[i]);
        }
    return s;
}

__device__ void finalize_epoch(KlCtl* ctl, uint32_t len, unsigned long long j, const EpochStats& S) {
    __threadfence();
    volatile KlFin* vf = &ctl->fin;
    KlFin F;
    F.rec = vf->rec;
    F.counters = vf->counters;
    F.tag = vf->tag;
    F.n_sms = vf->n_sms;
    const unsigned long long w = atomicAdd(&ctl->word, 0ull);
    // every id below min(next, limit) was handed out and executed by a block that has left;
    // over-fetched ids (>= limit) are discarded
    const uint32_t lim = min(word_limit(w, len), kl_w_next(w));
    const uint32_t mx = S.mx, executed = S.executed, admitted = S.admitted;
    const unsigned long long t0 = S.t0;
    const unsigned long long t1 = gtimer();
    const uint32_t start = ctl->base;
    ctl->base = lim;
    const bool exh = (lim == len);
    // next epoch: next = lim, stop cleared; membership reopened only if blocks remain (an
    // exhausted kernel's word stays closed, so no late block can ever open a phantom epoch)
    const uint32_t tk = kl_j_ticket(j);
    const uint32_t ne = kl_w_epoch(w) + 1u;
    atomicExch(&ctl->word, kl_w_make(lim, 0u, ne, false));
    __threadfence();
    if (!exh) {
        // reopen for the next epoch; the count is preserved (a late block's stray join may still
        // be pending its undo)
        unsigned long long cur = atomicAdd(&ctl->join, 0ull);
        for (;;) {
            const unsigned long long nw = (cur & 0xffffffffull) | kl_j_make((tk & ~0x7fu) | (ne & 0x7fu), false);
            const unsigned long long prev = atomicCAS(&ctl->join, cur, nw);
            if (prev == cur) break;
            cur = prev;
        }
    }
    if (F.counters) {
        atomicAdd(&F.counters[1], (unsigned long long)executed);
        if (exh) {
            atomicAdd(&F.counters[0], 1ull);
            atomicAdd(&F.counters[4], F.tag);
        }
        if (admitted) atomicMin(reinterpret_cast<long long*>(&F.counters[2]), (long long)t0);
        atomicMax(reinterpret_cast<long long*>(&F.counters[3]), (long long)t1);
    }
    KlLaunchRec* r = F.rec;
    if (r) {
#ifdef KL_PROBE_ANATOMY
        r->t_done = gtimer();
#endif
        r->start = start;
        r->end = lim;
        r->exhausted = exh ? 1u : 0u;
        r->executed = executed;
        r->admitted = admitted;
        r->max_per_sm = mx;
        r->t0 = t0;
        r->t1 = t1;
        __threadfence_system();
        r->done = 1u;
        __threadfence_system();
    }
}

// Leave the epoch; the block that brings the count to zero closes and finalizes it once its range
// is finished (exhausted, or stopped and drained to the boundary).
// Leave the epoch; true (and the membership word through *jout) if this block closed it -- the
// caller then finalizes.
__device__ bool leave_epoch_try(KlCtl* ctl, unsigned long long* jout) {
    __threadfence();
    const unsigned long long j = atomicAdd(&ctl->join, ~0ull) - 1ull;   // count - 1
    if (kl_j_count(j) != 0 || kl_j_closed(j)) return false;
    const uint32_t len = ctl->len;
    const unsigned long long w = atomicAdd(&ctl->word, 0ull);
    if (kl_w_next(w) < word_limit(w, len)) return false;   // not finished: live blocks will come
    if (atomicCAS(&ctl->join, j, j | KL_J_CLOSED) != j) return false;
    *jout = j;
    return true;
}

// Single-thread leave (a late block undoing a stray join): finalizes serially if it closes.
__device__ void leave_epoch(KlCtl* ctl) {
    unsigned long long j;
    if (leave_epoch_try(ctl, &j)) finalize_epoch(ctl, ctl->len, j, gather_stats_serial(ctl, ctl->fin.n_sms));
}

// Join the grid's epoch (false: closed, another epoch, or a recycled slot -> exit untouched).
__device__ bool join_epoch(const KlLaunch& L) {
    KlCtl* ctl = L.ctl;
    const unsigned long long j0 = *(volatile unsigned long long*)&ctl->join;
    if (kl_j_closed(j0) || kl_j_ticket(j0) != L.ticket) return false;   // late block: no atomics
    const unsigned long long j = atomicAdd(&ctl->join, 1ull);
    if (kl_j_closed(j) || kl_j_ticket(j) != L.ticket) {
        // raced with a close/reopen: undo the stray count (and close if it was the last)
        leave_epoch(ctl);
        return false;
    }
    KlFin* f = &ctl->fin;
    if (f->rec != L.rec) f->rec = L.rec;
    if (f->counters != L.counters) f->counters = L.counters;
    if (f->tag != L.tag) f->tag = L.tag;
    if (f->n_sms != L.n_sms) f->n_sms = L.n_sms;
    __threadfence();
    return true;
}

// Occupancy cap in force for this grid's epoch: the host re-tune if it names the epoch, else the
// grid's own cap (0 = uncapped).
__device__ __forceinline__ uint32_t cap_now(const KlLaunch& L, const KlCtl* ctl) {
    const unsigned long long t = ctl->tune;
    if ((t & 1ull) && ((t >> 1) & 0x7full) == (L.ticket & 0x7fu)) return (uint32_t)(t >> 32);
    return L.cap;
}

// Optional Body::kMinBlocks: resident blocks per SM the register allocation must allow (keeps
// the persistent variant at the plain kernel's occupancy despite the fetch logic).
template <class B, class = void>
struct min_blocks { static constexpr int value = 0; };   // 0 = unspecified
template <class B>
struct min_blocks<B, std::void_t<decltype(B::kMinBlocks)>> { static constexpr int value = B::kMinBlocks; };

// Optional Body::block_range(P, st, dsmem, v0, v1): the body runs a fetched chunk of virtual
// blocks [v0, v1) together (more independent work in flight per block: SPMV's rows); the
// per-block result must not depend on how the range is grouped (sliced == unsliced).  Such a
// body needs no Body::block.
template <class B, class = void>
struct has_range : std::false_type {};
template <class B>
struct has_range<B, std::void_t<decltype(&B::block_range)>> : std::true_type {};

template <class Body>
__global__ void __launch_bounds__(Body::kThreads, min_blocks<Body>::value)
k_persistent(const __grid_constant__ typename Body::Params P, const __grid_constant__ KlLaunch L) {
    extern __shared__ __align__(1024) char dsmem[];
    __shared__ uint32_t s_vb[2], s_end[2], s_adm;
#ifdef KL_PROBE_ANATOMY
    if (blockIdx.x == 0 && threadIdx.x == 0 && L.rec) L.rec->t_entry = gtimer();
#endif
    KlCtl* ctl = L.ctl;
    const uint32_t len = ctl->len;
    uint32_t sm = 0;
    bool joined = false;
    if (threadIdx.x == 0) {
        uint32_t adm = 0;
        joined = join_epoch(L);
        if (joined) {
            sm = smid_u32();
            const uint32_t cap = cap_now(L, ctl);
            const uint32_t c = atomicAdd(&ctl->sm_count[sm], 1u);
            if (cap && c >= cap) {
                atomicSub(&ctl->sm_count[sm], 1u);
            } else {
                adm = 1;
                atomicMax(&ctl->sm_hwm[sm], c + 1);
                atomicAdd(&ctl->sm_adm[sm], 1u);
                const unsigned long long now = gtimer();
                if (atomicCAS(&ctl->sm_t0[sm], 0ull, now) != 0ull) atomicMin(&ctl->sm_t0[sm], now);
            }
        }
        s_adm = adm;
    }
    __syncthreads();
    if (s_adm) {
        typename Body::State st;
        Body::init(P, st, dsmem);
        uint32_t nexec = 0;
        bool counted = true;   // this block still holds an sm_count slot
        for (uint32_t it = 0;; ++it) {
            if (threadIdx.x == 0) {
                uint32_t vb = 0, end = 0;
                // occupancy lowered by a re-tune: surplus blocks on this SM leave (no fetch)
                const uint32_t cap = cap_now(L, ctl);
                bool leave = false;
                if (cap) {
                    uint32_t c = *(volatile uint32_t*)&ctl->sm_count[sm];
                    while (c > cap) {
                        const uint32_t prev = atomicCAS(&ctl->sm_count[sm], c, c - 1u);
                        if (prev == c) { leave = true; counted = false; break; }
                        c = prev;
                    }
                }
                if (!leave) {
                    const unsigned long long req = ctl->stop_req;
                    unsigned long long old = atomicAdd(&ctl->word, (unsigned long long)L.chunk);
                    if ((req & 1ull) && !(old & KL_W_STOP) && ((req >> 1) & 0x7full) == kl_w_epoch(old)) {
                        // a host re-plan asked this epoch to stop: set the boundary (>= this fetch)
                        stop_word(ctl, kl_w_epoch(old), (uint32_t)(req >> 32));
                        old = (atomicAdd(&ctl->word, 0ull) & ~KL_W_MASK28) | (old & KL_W_MASK28);
                    }
                    vb = kl_w_next(old);
                    const uint32_t lim = word_limit(old, len);
                    end = vb < lim ? min(vb + L.chunk, lim) : vb;
                    if (vb >= len && lim == len && L.rec) {
                        // the kernel has no more thread blocks: raise the drained event once
                        if (atomicCAS(&ctl->drained, 0u, 1u) == 0u) {
                            L.rec->drained = 1u;
                            __threadfence_system();
                        }
                    }
                }
                s_vb[it & 1] = vb;
                s_end[it & 1] = end;
            }
            __syncthreads();
            const uint32_t vb = s_vb[it & 1], end = s_end[it & 1];
            if (vb >= end) break;
            if constexpr (has_range<Body>::value) {
                const unsigned long long t_a = (L.stamps && threadIdx.x == 0) ? gtimer() : 0ull;
                Body::block_range(P, st, dsmem, vb, end);
                if (threadIdx.x == 0) {
                    const unsigned long long t_b = L.stamps ? gtimer() : 0ull;
                    for (uint32_t v = vb; v < end; ++v) {
                        if (L.audit) atomicAdd(L.audit + v, 1u);
                        if (L.stamps) { L.stamps[2 * (size_t)v] = t_a; L.stamps[2 * (size_t)v + 1] = t_b; }
                    }
                }
            } else {
                for (uint32_t v = vb; v < end; ++v) {
                    if (L.stamps && threadIdx.x == 0) L.stamps[2 * (size_t)v] = gtimer();
                    Body::block(P, st, dsmem, v);
                    if (L.audit && threadIdx.x == 0) atomicAdd(L.audit + v, 1u);
                    if (L.stamps && threadIdx.x == 0) L.stamps[2 * (size_t)v + 1] = gtimer();
                }
            }
            nexec += end - vb;
        }
        Body::fini(P, st, dsmem);
        if (threadIdx.x == 0) {
            atomicAdd(&ctl->sm_exec[sm], nexec);
            if (counted) atomicSub(&ctl->sm_count[sm], 1u);
        }
    }
    // leave; the block whose leave closes the epoch finalizes it, gathering the per-SM statistics
    // with all its threads
    __shared__ int s_close;
    __shared__ unsigned long long s_j;
    if (threadIdx.x == 0) {
        unsigned long long j = 0ull;
        s_close = (joined && leave_epoch_try(ctl, &j)) ? 1 : 0;
        s_j = j;
    }
    __syncthreads();
    if (s_close) {
        const EpochStats S = gather_stats_block<Body::kThreads>(ctl, L.n_sms);
        if (threadIdx.x == 0) finalize_epoch(ctl, len, s_j, S);
    }
}

// ---- CTA pairs (thread-block clusters of 2 on one TPC) ------------------------------------
// A body with kPair = true runs one virtual block on a CTA pair (tcgen05 cta_group::2: the two
// SMs' tensor cores compute one tile from operands split across their shared memories).  The
// pair joins, is admitted and fetches as ONE unit: each CTA passes its own SM's admission cap,
// the leader (cluster rank 0) fetches and hands the range to its peer through distributed shared
// memory, and both run Body::block on the same virtual block.  Statistics (executed blocks,
// audit, stamps) are the leader's.
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `local` (a shared::cta address) in the CTA of cluster rank `rank`
__device__ __forceinline__ uint32_t map_rank(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// Optional Body::kRun + Body::run(P, st, dsmem, fetcher, L): the pair body owns its tile loop
// (its roles synchronise through mbarriers instead of one CTA + one cluster barrier per tile)
// and calls fetcher.next() -- on the leader's thread 0 only -- whenever it wants the next
// virtual block; next() returns (vb << 2) | part, or 0xFFFFFFFF when the pair is done.
template <class B, class = void>
struct has_run : std::false_type {};
template <class B>
struct has_run<B, std::void_t<decltype(B::kRun)>> : std::integral_constant<bool, B::kRun> {};

// The persistent launcher's fetch (leave on a lowered cap, stop requests, the drained event),
// one virtual block at a time out of the fetched chunk; stamps the start of each block.
struct PairFetcher {
    const KlLaunch* L;
    KlCtl* ctl;
    uint32_t len, sm, cur, end, nexec;
    bool counted, done;
    __device__ uint32_t next() {
        if (done) return 0xFFFFFFFFu;
        if (cur >= end) {
            const uint32_t cap = cap_now(*L, ctl);
            if (cap) {
                uint32_t c = *(volatile uint32_t*)&ctl->sm_count[sm];
                while (c > cap) {
                    const uint32_t prev = atomicCAS(&ctl->sm_count[sm], c, c - 1u);
                    if (prev == c) { counted = false; done = true; return 0xFFFFFFFFu; }
                    c = prev;
                }
            }
            const unsigned long long req = ctl->stop_req;
            unsigned long long old = atomicAdd(&ctl->word, (unsigned long long)L->chunk);
            if ((req & 1ull) && !(old & KL_W_STOP) && ((req >> 1) & 0x7full) == kl_w_epoch(old)) {
                stop_word(ctl, kl_w_epoch(old), (uint32_t)(req >> 32));
                old = (atomicAdd(&ctl->word, 0ull) & ~KL_W_MASK28) | (old & KL_W_MASK28);
            }
            const uint32_t vb = kl_w_next(old);
            const uint32_t lim = word_limit(old, len);
            if (vb >= len && lim == len && L->rec) {
                if (atomicCAS(&ctl->drained, 0u, 1u) == 0u) {
                    L->rec->drained = 1u;
                    __threadfence_system();
                }
            }
            if (vb >= lim) { done = true; return 0xFFFFFFFFu; }
            cur = vb;
            end = min(vb + L->chunk, lim);
        }
        const uint32_t v = cur++;
        ++nexec;
        if (L->stamps) L->stamps[2 * (size_t)v] = gtimer();
        return v << 2;
    }
};

// The plain pair grid's static schedule: cluster c takes offset + c, c + n_clusters, ... and, when
// the last round would leave more than half the pairs idle, half tiles of the remainder.
struct StaticPairFetcher {
    uint32_t offset, c, ncl, full, rem, i;
    bool split;
    __device__ uint32_t next() {
        const uint32_t v = c + i * ncl;
        ++i;
        if (v < full) return (offset + v) << 2;
        if (split && v - full < ncl && c < 2 * rem && v - full == c)   // the one half-tile item
            return ((offset + full + c / 2) << 2) | (1u + (c & 1u));
        return 0xFFFFFFFFu;
    }
};

template <class Body>
__global__ void __cluster_dims__(2, 1, 1) __maxnreg__(64)
k_persistent_pair(const __grid_constant__ typename Body::Params P, const __grid_constant__ KlLaunch L) {
    extern __shared__ __align__(1024) char dsmem[];
    __shared__ uint32_t s_vb[2], s_end[2], s_adm, s_peer_adm;
    KlCtl* ctl = L.ctl;
    const uint32_t len = ctl->len;
    const uint32_t rank = cluster_rank();
    uint32_t sm = 0;
    bool joined = false;
    // distributed shared memory may only be written once the peer CTA is running
    // (compute-sanitizer: "a block that might not have entered yet")
    cluster_sync_all();
    if (threadIdx.x == 0) {
        uint32_t adm = 0;
        joined = join_epoch(L);
        if (joined) {
            sm = smid_u32();
            const uint32_t cap = cap_now(L, ctl);
            const uint32_t c = atomicAdd(&ctl->sm_count[sm], 1u);
            if (cap && c >= cap) atomicSub(&ctl->sm_count[sm], 1u);
            else adm = 1;
        }
        s_adm = adm;
        st_cluster_u32(map_rank(smem_u32_of(&s_peer_adm), rank ^ 1u), adm);
    }
    cluster_sync_all();
    const bool pair_ok = s_adm && s_peer_adm;
    if (threadIdx.x == 0 && s_adm) {
        if (!pair_ok) {
            atomicSub(&ctl->sm_count[sm], 1u);     // the peer was refused: release this SM's slot
        } else {
            const uint32_t c = *(volatile uint32_t*)&ctl->sm_count[sm];
            atomicMax(&ctl->sm_hwm[sm], c);
            atomicAdd(&ctl->sm_adm[sm], 1u);
            const unsigned long long now = gtimer();
            if (atomicCAS(&ctl->sm_t0[sm], 0ull, now) != 0ull) atomicMin(&ctl->sm_t0[sm], now);
        }
    }
    if (pair_ok) {
        typename Body::State st;
        Body::init(P, st, dsmem);
        uint32_t nexec = 0;
        bool counted = true;
        if constexpr (has_run<Body>::value) {
            PairFetcher f{&L, ctl, len, sm, 0u, 0u, 0u, true, false};
            Body::run(P, st, dsmem, f, &L);
            if (threadIdx.x == 0 && rank == 0) { nexec = f.nexec; counted = f.counted; }
        } else
        for (uint32_t it = 0;; ++it) {
            if (threadIdx.x == 0 && rank == 0) {
                uint32_t vb = 0, end = 0;
                const uint32_t cap = cap_now(L, ctl);
                bool leave = false;
                if (cap) {
                    uint32_t c = *(volatile uint32_t*)&ctl->sm_count[sm];
                    while (c > cap) {
                        const uint32_t prev = atomicCAS(&ctl->sm_count[sm], c, c - 1u);
                        if (prev == c) { leave = true; counted = false; break; }
                        c = prev;
                    }
                }
                if (!leave) {
                    const unsigned long long req = ctl->stop_req;
                    unsigned long long old = atomicAdd(&ctl->word, (unsigned long long)L.chunk);
                    if ((req & 1ull) && !(old & KL_W_STOP) && ((req >> 1) & 0x7full) == kl_w_epoch(old)) {
                        stop_word(ctl, kl_w_epoch(old), (uint32_t)(req >> 32));
                        old = (atomicAdd(&ctl->word, 0ull) & ~KL_W_MASK28) | (old & KL_W_MASK28);
                    }
                    vb = kl_w_next(old);
                    const uint32_t lim = word_limit(old, len);
                    end = vb < lim ? min(vb + L.chunk, lim) : vb;
                    if (vb >= len && lim == len && L.rec) {
                        if (atomicCAS(&ctl->drained, 0u, 1u) == 0u) {
                            L.rec->drained = 1u;
                            __threadfence_system();
                        }
                    }
                }
                s_vb[it & 1] = vb;
                s_end[it & 1] = end;
                st_cluster_u32(map_rank(smem_u32_of(&s_vb[it & 1]), 1u), vb);
                st_cluster_u32(map_rank(smem_u32_of(&s_end[it & 1]), 1u), end);
            }
            Body::before_pair_sync(st);
            cluster_sync_all();   // the range is visible to the peer; both finished the previous tile
            Body::after_pair_sync(st);
            const uint32_t vb = s_vb[it & 1], end = s_end[it & 1];
            if (vb >= end) break;
            for (uint32_t v = vb; v < end; ++v) {
                if (rank == 0 && L.stamps && threadIdx.x == 0) L.stamps[2 * (size_t)v] = gtimer();
                Body::block(P, st, dsmem, v);
                if (rank == 0 && L.audit && threadIdx.x == 0) atomicAdd(L.audit + v, 1u);
                if (rank == 0 && L.stamps && threadIdx.x == 0) L.stamps[2 * (size_t)v + 1] = gtimer();
            }
            nexec += end - vb;
        }
        Body::fini(P, st, dsmem);
        if (threadIdx.x == 0) {
            if (rank == 0) atomicAdd(&ctl->sm_exec[sm], nexec);
            // the peer's slot: released unless the leader's cap check released the pair's (the
            // leader's decision to leave is the pair's; its peer's SM keeps the cap too)
            if (counted) atomicSub(&ctl->sm_count[sm], 1u);
        }
    }
    __shared__ int s_close;
    __shared__ unsigned long long s_j;
    if (threadIdx.x == 0) {
        unsigned long long j = 0ull;
        s_close = (joined && leave_epoch_try(ctl, &j)) ? 1 : 0;
        s_j = j;
    }
    __syncthreads();
    if (s_close) {
        const EpochStats S = gather_stats_block<Body::kThreads>(ctl, L.n_sms);
        if (threadIdx.x == 0) finalize_epoch(ctl, len, s_j, S);
    }
}

// Plain grid of CTA pairs: one resident pair per TPC, cluster c runs virtual blocks offset + c,
// offset + c + n_clusters, ... (a static tile loop: the pair's setup -- barriers, TMEM
// allocation -- and its epilogue overlap across its tiles instead of being paid per tile).
template <class Body>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Body::kThreads, 1)
k_plain_pair(const __grid_constant__ typename Body::Params P, uint32_t offset, uint32_t n) {
    extern __shared__ __align__(1024) char dsmem[];
    uint32_t ncl;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(ncl));
    cluster_sync_all();   // both CTAs running before the pair's TMEM allocation touches either
    typename Body::State st;
    Body::init(P, st, dsmem);
    const uint32_t c = cluster_id_x();
    // full rounds of one tile per pair; a last round that would leave more than half the pairs
    // idle is split into half tiles (Body::block_part) so that every pair gets work
    const uint32_t rounds = n / ncl, rem = n - rounds * ncl;
    const bool split = rem > 0 && 2 * rem <= ncl;
    const uint32_t full = split ? rounds * ncl : n;
    if constexpr (has_run<Body>::value) {
        StaticPairFetcher f{offset, c, ncl, full, rem, 0u, split};
        Body::run(P, st, dsmem, f, (const KlLaunch*)nullptr);
        Body::fini(P, st, dsmem);
        return;
    }
    bool first = true;
    for (uint32_t v = c; v < full; v += ncl) {
        if (!first) {                    // the previous tile's hand-off, as in the pair launcher
            Body::before_pair_sync(st);
            cluster_sync_all();
            Body::after_pair_sync(st);
        }
        first = false;
        Body::block(P, st, dsmem, offset + v);
    }
    if (split && c < 2 * rem) {
        if (!first) {
            Body::before_pair_sync(st);
            cluster_sync_all();
            Body::after_pair_sync(st);
        }
        Body::block_part(P, st, dsmem, offset + full + c / 2, 1 + (int)(c & 1u));
    }
    Body::fini(P, st, dsmem);
}

// Plain grid: blockIdx rectified by the slice offset.  A body with block_range
// runs kChunk virtual blocks per grid block (the same grouping as a persistent fetch).
template <class Body>
__global__ void __launch_bounds__(Body::kThreads)
k_plain(const __grid_constant__ typename Body::Params P, uint32_t offset, uint32_t n) {
    extern __shared__ __align__(1024) char dsmem[];
    typename Body::State st;
    Body::init(P, st, dsmem);
    if constexpr (has_range<Body>::value) {
        const uint32_t v0 = blockIdx.x * (uint32_t)Body::kChunk;
        Body::block_range(P, st, dsmem, offset + v0, offset + min(n, v0 + (uint32_t)Body::kChunk));
    } else {
        Body::block(P, st, dsmem, offset + blockIdx.x);
    }
    Body::fini(P, st, dsmem);
}

template <class Body>
int info_of(KlKindInfo* o) {
    cudaFuncAttributes fa;
    cudaError_t e;
    if (Body::kDynSmem > 48 * 1024) {
        e = cudaFuncSetAttribute(k_persistent<Body>, cudaFuncAttributeMaxDynamicSharedMemorySize, Body::kDynSmem);
        if (e != cudaSuccess) return (int)e;
        e = cudaFuncSetAttribute(k_plain<Body>, cudaFuncAttributeMaxDynamicSharedMemorySize, Body::kDynSmem);
        if (e != cudaSuccess) return (int)e;
    }
    e = cudaFuncGetAttributes(&fa, k_persistent<Body>);
    if (e != cudaSuccess) return (int)e;
    int nb = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_persistent<Body>, Body::kThreads, Body::kDynSmem);
    if (e != cudaSuccess) return (int)e;
    o->threads = Body::kThreads;
    o->dyn_smem = Body::kDynSmem;
    o->regs = fa.numRegs;
    o->static_smem = (int)fa.sharedSizeBytes;
    o->tmem_cols = 0;
    o->bmax = nb;
    o->default_chunk = Body::kChunk;
    return 0;
}

template <class Body>
int launch_persistent(const void* blob, const KlLaunch& L, uint32_t grid, void* stream) {
    const auto& P = *reinterpret_cast<const typename Body::Params*>(blob);
    k_persistent<Body><<<grid, Body::kThreads, Body::kDynSmem, (cudaStream_t)stream>>>(P, L);
    return (int)cudaGetLastError();
}

// CTA-pair bodies: one resident pair per TPC (one CTA per SM: the body's shared memory and the
// whole TMEM), attributes from the pair kernels.
template <class Body>
int info_of_pair(KlKindInfo* o) {
    cudaFuncAttributes fa;
    cudaError_t e;
    e = cudaFuncSetAttribute(k_persistent_pair<Body>, cudaFuncAttributeMaxDynamicSharedMemorySize, Body::kDynSmem);
    if (e != cudaSuccess) return (int)e;
    e = cudaFuncSetAttribute(k_plain_pair<Body>, cudaFuncAttributeMaxDynamicSharedMemorySize, Body::kDynSmem);
    if (e != cudaSuccess) return (int)e;
    e = cudaFuncGetAttributes(&fa, k_persistent_pair<Body>);
    if (e != cudaSuccess) return (int)e;
    o->threads = Body::kThreads;
    o->dyn_smem = Body::kDynSmem;
    o->regs = fa.numRegs;
    o->static_smem = (int)fa.sharedSizeBytes;
    o->tmem_cols = 0;
    o->bmax = 1;
    o->default_chunk = Body::kChunk;
    return 0;
}

// `grid` CTAs, rounded up to whole pairs.
template <class Body>
int launch_persistent_pair(const void* blob, const KlLaunch& L, uint32_t grid, void* stream) {
    const auto& P = *reinterpret_cast<const typename Body::Params*>(blob);
    grid = (grid + 1u) & ~1u;
    k_persistent_pair<Body><<<grid, Body::kThreads, Body::kDynSmem, (cudaStream_t)stream>>>(P, L);
    return (int)cudaGetLastError();
}

// n virtual blocks on min(n, n_sms / 2) pairs.
template <class Body>
int launch_plain_pair(const void* blob, uint32_t offset, uint32_t n, void* stream) {
    const auto& P = *reinterpret_cast<const typename Body::Params*>(blob);
    if (n == 0) return 0;
    static int n_sms = 0;
    if (!n_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, dev);
        if (n_sms < 2) n_sms = 2;
    }
    const uint32_t pairs = std::min(n, (uint32_t)(n_sms / 2));
    k_plain_pair<Body><<<2 * pairs, Body::kThreads, Body::kDynSmem, (cudaStream_t)stream>>>(P, offset, n);
    return (int)cudaGetLastError();
}

template <class Body>
int launch_plain(const void* blob, uint32_t offset, uint32_t n, void* stream) {
    const auto& P = *reinterpret_cast<const typename Body::Params*>(blob);
    if (n == 0) return 0;
    const uint32_t blocks = has_range<Body>::value ? (n + Body::kChunk - 1) / Body::kChunk : n;
    k_plain<Body><<<blocks, Body::kThreads, Body::kDynSmem, (cudaStream_t)stream>>>(P, offset, n);
    return (int)cudaGetLastError();
}

}  // namespace
