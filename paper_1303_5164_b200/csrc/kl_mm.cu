// kl_mm.cu -- MM ("Multiplying two dense matrices", 8192x2048 . 2048x2048) on the
// 5th-generation tensor cores, one CTA PAIR per output tile (product path).
//
// One virtual thread block = one 256x256 fp32 output tile computed by a CTA pair (a cluster of 2
// on one TPC; kl_launcher.cuh k_persistent_pair): tcgen05.mma.cta_group::2 (M=256, N=256, K=16)
// reads A's 256 rows as 128 rows from each CTA's shared memory and B's 256 columns as 128 rows
// of Bt from each, and accumulates CTA r's 128 rows in CTA r's TMEM.  The launchers run the
// decoupled tile loop (BodyMM::run; the per-tile block() path is kept for reference):
//   leader thread 0 : scheduler -- claims each tile from the launcher's fetch (or the plain grid's
//                   static schedule) when the leader's producer asks for it, and publishes it
//                   through a 4-deep tile-info ring in both CTAs' shared memory;
//   warp 2 lane 0 : TMA producer (both CTAs) -- its CTA's 128x64 (A) and 128x64 (B) bf16 tiles,
//                   128B swizzle, into a ring of S shared-memory stages, streaming across tile
//                   boundaries; completion (.cta_group::2) on the LEADER's full barrier;
//   warp 1 lane 0 : MMA issuer (leader only) -- waits for a drained accumulator (tempty), then 4
//                   MMAs per stage into one of two 256-column fp32 accumulators; tcgen05.commit
//                   multicast frees the stage in both CTAs and, after the last k-block, signals
//                   both CTAs' epilogues;
//   warps 4..7    : epilogue (both CTAs) -- drain the previous tile's accumulator (tcgen05.ld
//                   32x32b.x32, each warp its 32 TMEM lanes) through a swizzled shared-memory box
//                   into coalesced 128-byte STG lines while the next tile's mainloop runs.
// Against one-CTA 128x256 tiles this halves the operand bytes each SM pulls from L2 per MMA
// (the one-CTA kernel is L2-feed-bound at 48 % of the bf16 peak).
// The stage count S in {2, 3, 4, 6} (32 KiB of shared memory each) is the kernel's occupancy
// knob: MM's occupancy levels; one instantiation per level.
// Numerics: bf16 products are exact in fp32; only the fp32 accumulation order differs from the
// oracle's fp64 sum (normwise tolerance).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <algorithm>
#include <cstring>
#include "kl_internal.h"
#include "kl_launcher.cuh"

namespace {

constexpr int BM = 128;            // A rows per CTA (the pair's tile is 2*BM = 256 rows)
constexpr int BN = 256;            // tile columns (the pair's N)
constexpr int BNH = BN / 2;        // Bt rows per CTA
constexpr int BK = 64;             // k per stage (one 128-byte swizzle atom of bf16)
constexpr int kStageBytes = (BM + BNH) * BK * 2;   // 32 KiB per CTA
constexpr int kThreads = 256;      // 8 warps: whole warps per virtual SM (R14)
constexpr uint32_t kTmemCols = 2 * BN;             // two fp32 accumulators (tile i / epilogue of i-1)
// instruction descriptor: F32 accumulate, BF16 A/B, K-major A/B, N = 256, M = 256 (pair)
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
constexpr uint32_t kIdescHalf = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)((BN / 2) >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
constexpr int kStageLevels[4] = {2, 3, 4, 6};

constexpr int kEpiBox = 32;                        // C store box: 32 rows x 32 fp32 (128 B rows)
constexpr int kEpiBufBytes = kEpiBox * kEpiBox * 4;  // 4 KiB
constexpr int kEpiBytes = 4 * 2 * kEpiBufBytes;      // 4 epilogue warps x 2 buffers
// Barrier block (offsets from State::bars): full[s] 0+8s, empty[s] 64+8s, tfull[b] 128+8b,
// tempty[b] 144+8b, tile-info full[q] 160+8q, TMEM base address 192, need-next 200,
// tile-info empty[q] 256+8q, tile-info slots (u32) 320+4q.
constexpr int kBarBytes = 512;
constexpr int kTileQ = 4;                            // tile-info ring depth (run loop)
constexpr uint32_t kItemNone = 0xFFFFFFFFu;          // end of the pair's tile sequence
// tile-info consumers: producer + MMA issuer + 4 epilogue warps (CTA 0), producer + 4 epilogue
// warps (CTA 1)
constexpr uint32_t kTileConsumers = 11;

struct MMParams {
    CUtensorMap ta;   // A  [M][K] bf16, box 64 x 128
    CUtensorMap tb;   // Bt [N][K] bf16, box 64 x 128
    CUtensorMap tbh;  // Bt [N][K] bf16, box 64 x 64 (half-width tiles, the plain grid's tail)
    CUtensorMap tc;   // C  [M][N] fp32, box 32 x 32, 128B swizzle (TMA store epilogue)
    float* C;
    int32_t M, N, K;
};
static_assert(sizeof(MMParams) <= 1024, "blob");

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#ifdef KL_MM_PROBE
// Timing probe (tools/mm_stamp_probe.py; not in the product build): per pair (cluster id) and per
// tile j < 8: [0] MMA issuer sees the first stage full, [1] last MMA of the tile issued,
// [2] epilogue (rank 0, warp 4) starts waiting for the accumulator, [3] its TMA stores issued;
// per pair [kProbeTiles*4] kernel entry, [+1] after init, [+2] before fini, [+3] end of fini.
constexpr int kProbeTiles = 8, kProbeF = 8, kProbeStride = kProbeTiles * kProbeF + 4;
__device__ unsigned long long g_mm_probe[96 * kProbeStride];
__device__ __forceinline__ unsigned long long probe_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t probe_cluster() {
    uint32_t c;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(c));
    return c;
}
#define MM_PROBE(j, f) do { const uint32_t c_ = probe_cluster(); if (c_ < 96 && (j) < kProbeTiles) g_mm_probe[c_ * kProbeStride + (j) * kProbeF + (f)] = probe_now(); } while (0)
#define MM_PROBE_K(f) do { const uint32_t c_ = probe_cluster(); if (c_ < 96) g_mm_probe[c_ * kProbeStride + kProbeTiles * kProbeF + (f)] = probe_now(); } while (0)
#define MM_PROBE_T(f) do { if (probe_tile < kProbeTiles) MM_PROBE(probe_tile, f); } while (0)
#else
#define MM_PROBE_T(f) do { } while (0)
#define MM_PROBE(j, f) do { } while (0)
#define MM_PROBE_K(f) do { } while (0)
#endif

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// Waits whose barrier receives arrivals from the peer CTA (acquire at cluster scope: the peer's
// shared::cluster writes before its release-arrive are visible after the wait).
__device__ __forceinline__ void mbar_wait_cl(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// Arrive on this CTA's barrier with CTA-scope release.  Not cluster scope: a cluster-scope
// release issued by the MMA thread waits for its outstanding tcgen05 MMAs (device stamps,
// tools/mm_stamp_probe.py: ~1.8 us per tile boundary -- the same stall the per-tile
// barrier.cluster.arrive.release of the block() path pays).
__device__ __forceinline__ void mbar_arrive_local(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// arrive on the barrier at shared::cluster address `bar_cl` (this CTA's or the peer's)
__device__ __forceinline__ void mbar_arrive_cl(uint32_t bar_cl) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cl) : "memory");
}
// TMA 2-D load into this CTA's shared memory; completion bytes land on `bar_cluster` (a
// shared::cluster address: the leader CTA's full barrier).
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                 int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"((uint64_t)map), "r"(bar_cluster), "r"(c0), "r"(c1)
        : "memory");
}
// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row core groups 1024 B apart.
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr & 0x3FFFFu) >> 4);        // start address  [0,14)
    d |= (uint64_t)1 << 16;                         // LBO (unused for swizzled K-major) [16,30)
    d |= (uint64_t)(1024 >> 4) << 32;               // SBO = 1024 B  [32,46)
    d |= (uint64_t)1 << 46;                         // version = 1 (sm_100)
    d |= (uint64_t)2 << 61;                         // SWIZZLE_128B
    return d;
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
// Arrive on the barrier at shared offset `bar` in both CTAs of the pair once the MMAs issued so
// far complete.
__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(bar)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

#define TMEM_LD_X32(taddr, r)                                                                                 \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 "                                                   \
                 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24," \
                 "%25,%26,%27,%28,%29,%30,%31}, [%32];"                                                        \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),      \
                   "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),  \
                   "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),            \
                   "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),            \
                   "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])             \
                 : "r"(taddr))

template <int S>
struct BodyMM {
    static_assert(S >= 2 && S <= 6, "stages");
    using Params = MMParams;
    static constexpr int kThreads = ::kThreads, kChunk = 1;
    static constexpr int kDynSmem = S * kStageBytes + kEpiBytes + 1024 /*align*/ + kBarBytes;
    static constexpr int kEpiOffset = S * kStageBytes;
    static constexpr int kBarOffset = S * kStageBytes + kEpiBytes;
    struct State {
        uint32_t base;      // 1024-aligned shared address of stage 0
        uint32_t bars;      // full[s] bars+8s, empty[s] bars+64+8s, tfull[b] bars+128+8b, tmem ptr bars+192
        uint32_t tmem;
        uint32_t rank;      // rank in the CTA pair (0: leader, issues the MMAs)
        uint32_t stage, phase;
        uint32_t tph;       // per-accumulator wait parity bits
        uint32_t ntile;     // tiles issued by this persistent pair
        int prev_m, prev_col, prev_w; // tile whose accumulator is still to be drained (-1: none):
                                      // row tile, first column, width
    };
    __device__ static void init(const Params&, State& st, char* dsmem) {
        const uint32_t raw = smem_u32(dsmem);
        if (threadIdx.x == 0 && cluster_rank() == 0) MM_PROBE_K(0);
        st.base = (raw + 1023u) & ~1023u;
        st.bars = st.base + kBarOffset;
        st.rank = cluster_rank();
        st.stage = st.phase = st.tph = st.ntile = 0;
        st.prev_m = st.prev_col = -1;
        st.prev_w = BN;
        const int warp = threadIdx.x >> 5;
        if (threadIdx.x == 0) {
            for (int s = 0; s < S; ++s) {
                mbar_init(st.bars + 8 * s, 1);
                mbar_init(st.bars + 64 + 8 * s, 1);
            }
            mbar_init(st.bars + 128, 1);
            mbar_init(st.bars + 136, 1);
            mbar_init(st.bars + 144, 8);     // tempty[b]: the 4 epilogue warps of both CTAs drained b
            mbar_init(st.bars + 152, 8);
            mbar_init(st.bars + 200, 1);     // need-next: the leader's producer asks for the next tile
            for (int q = 0; q < kTileQ; ++q) {
                mbar_init(st.bars + 160 + 8 * q, 1);
                mbar_init(st.bars + 256 + 8 * q, kTileConsumers);
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        if (warp == 1) {   // the same warp in both CTAs allocates the pair's columns
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(st.bars + 192),
                         "r"(kTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        }
        tc_fence_before();
        cluster_sync_all();   // barriers initialised and TMEM allocated in both CTAs
        __syncthreads();      // (also a CTA barrier for racecheck, which does not model the cluster one)
        tc_fence_after();
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(st.tmem) : "r"(st.bars + 192));
        if (threadIdx.x == 0 && st.rank == 0) MM_PROBE_K(1);
    }
    __device__ static void before_pair_sync(State&) { tc_fence_before(); }
    __device__ static void after_pair_sync(State&) { tc_fence_after(); }
    // Epilogue warps: wait for tile (m, n)'s accumulator b and move this CTA's 128 rows TMEM ->
    // registers -> shared memory (128B-swizzled 32x32 boxes, two buffers per warp) -> C by TMA
    // bulk-tensor stores (whole 128-byte lines; a thread-per-row STG epilogue issues 32 partial
    // sectors per instruction and was the launch's tail).
    __device__ static void drain(const Params& P, State& st, int m, int col, int w, uint32_t b) {
        drain_tile(P, st, m, col, w, b, (st.tph >> b) & 1u, st.ntile - 1);
        if ((threadIdx.x >> 5) == 4 && (threadIdx.x & 31) == 0 && st.rank == 0) MM_PROBE(st.ntile - 1, 3);
    }
    __device__ static void drain_tile(const Params& P, State& st, int m, int col, int w, uint32_t b, uint32_t parity,
                                      uint32_t probe_tile = 0xFFFFu) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        mbar_wait(st.bars + 128 + 8 * b, parity);
        if (warp == 4 && lane == 0 && st.rank == 0) MM_PROBE_T(2);
        tc_fence_after();
        const int q = warp & 3;                              // TMEM lane quarter of this warp
        const int row0 = m * (2 * BM) + (int)st.rank * BM + q * 32;
        const uint32_t tbase = st.tmem + ((uint32_t)(q * 32) << 16) + b * BN;
        const uint32_t ebuf = st.base + kEpiOffset + (uint32_t)q * 2u * kEpiBufBytes;
#pragma unroll 1
        for (int c = 0; c < w; c += 32) {
            uint32_t r[32];
            TMEM_LD_X32(tbase + (uint32_t)c, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const uint32_t buf = ebuf + (uint32_t)((c >> 5) & 1) * kEpiBufBytes;
#ifdef KL_MM_EPI_TMA
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");   // buf's last store read it
#endif
            __syncwarp();
#ifdef KL_MM_DBG_NOEPI      // A/B probe: no C stores
            if (r[0] == 0x7fffffffu && r[1] == 0x7fffffffu)
#endif
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t a = buf + (uint32_t)lane * 128u + (uint32_t)((j ^ (lane & 7)) * 16);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(r[4 * j]), "r"(r[4 * j + 1]),
                             "r"(r[4 * j + 2]), "r"(r[4 * j + 3])
                             : "memory");
            }
#ifdef KL_MM_EPI_TMA
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                asm volatile(
                    "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"((uint64_t)&P.tc),
                    "r"(buf), "r"(col + c), "r"(row0)
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
#else
            // coalesced stores from the staged 32x32 box: 8 lanes per 128-byte row, 4 rows per
            // instruction (whole lines; no TMA store queued behind the operand loads, no bulk-group
            // wait before the buffer's reuse -- the accumulator frees at the TMEM-load rate)
            __syncwarp();
            {
                const int seg = lane & 7;
                float* cbase = P.C + (size_t)row0 * (size_t)P.N + (size_t)(col + c) + (size_t)seg * 4;
#pragma unroll
                for (int it = 0; it < 8; ++it) {
                    const int row = it * 4 + (lane >> 3);
                    const uint32_t a = buf + (uint32_t)row * 128u + (uint32_t)((seg ^ (row & 7)) * 16);
                    uint32_t v0, v1, v2, v3;
                    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3) : "r"(a));
                    float* g = cbase + (size_t)row * (size_t)P.N;
                    asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(g), "r"(v0), "r"(v1), "r"(v2), "r"(v3)
                                 : "memory");
                }
            }
#endif
        }
        tc_fence_before();
    }
    __device__ static void fini(const Params& P, State& st, char*) {
        if (threadIdx.x == 0 && st.rank == 0) MM_PROBE_K(2);
        if (st.prev_m >= 0 && (threadIdx.x >> 5) >= 4) drain(P, st, st.prev_m, st.prev_col, st.prev_w, (st.ntile - 1) & 1u);
#ifdef KL_MM_EPI_TMA
        if ((threadIdx.x >> 5) >= 4 && (threadIdx.x & 31) == 0)
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // C written before the kernel's end
#endif
        tc_fence_before();
        cluster_sync_all();   // both CTAs drained: the pair's columns can go
        tc_fence_after();
        if ((threadIdx.x >> 5) == 1)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(st.tmem), "r"(kTmemCols));
        if (threadIdx.x == 0 && st.rank == 0) MM_PROBE_K(3);
    }
    // ---- decoupled tile loop (the launchers' Body::run path) ---------------------------------
    // The pair's roles run their own loops over the pair's tile sequence, synchronised only by
    // mbarriers: the leader's producer takes each tile from `f` (the launcher's fetch, or the
    // plain grid's static schedule) as soon as it has issued the previous tile's last operand
    // load, publishes it through a 4-deep tile-info ring in both CTAs' shared memory, and keeps
    // streaming operands into the ring of stages across the tile boundary; the MMA issuer waits
    // for an accumulator only until both CTAs' epilogues released it (tempty); the epilogue of
    // tile i overlaps the mainloop of tile i+1.  Against the per-tile block() (one CTA barrier and
    // one cluster barrier per tile, the producer idle until both) this removes the ~2.2 us gap
    // between a tile's last MMA and the next tile's first full stage (tools/mm_stamp_probe.py).
    // Item = (virtual block << 2) | part (0: 256x256 tile, 1 / 2: its left / right 256x128 half).
    static constexpr bool kRun = true;
    __device__ static uint32_t tile_item(State& st, uint32_t i) {   // consumer side of the tile-info ring
        const uint32_t q = i % kTileQ;
        mbar_wait_cl(st.bars + 160 + 8 * q, (i / kTileQ) & 1u);
        uint32_t item;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(item) : "r"(st.bars + 320 + 4 * q) : "memory");
        return item;
    }
    __device__ static void tile_release(State& st, uint32_t i) {   // one arrival per consumer
        const uint32_t bar = st.bars + 256 + 8 * (i % kTileQ);
        if (st.rank == 0) mbar_arrive_local(bar);
        else mbar_arrive_cl(map_rank(bar, 0u));
    }
    __device__ static void load_tile(const Params& P, State& st, uint32_t item, uint32_t probe_i = 0xFFFFu) {   // producer lanes
        const uint32_t vb = item >> 2;
        const int part = (int)(item & 3u);
        const int tiles_n = P.N / BN;
        const int tm = (int)vb / tiles_n, tn = (int)vb % tiles_n;
        const int nk = P.K / BK;
        const int w = part ? BN / 2 : BN;
        const int col = tn * BN + (part == 2 ? BN / 2 : 0);
        const CUtensorMap* tmb = part ? &P.tbh : &P.tb;
        const uint32_t tx = 2u * (uint32_t)(BM * BK * 2 + (w / 2) * BK * 2);
        const int arow = tm * (2 * BM) + (int)st.rank * BM, brow = col + (int)st.rank * (w / 2);
        const int kneed = nk > S ? nk - S : 0;
        for (int kb = 0; kb < nk; ++kb) {
            // the leader asks for the next tile S stages before this one's last load, so the
            // scheduler's fetch overlaps the loads still to come (a just-in-time claim)
            if (kb == kneed && st.rank == 0) mbar_arrive_local(st.bars + 200);
            mbar_wait(st.bars + 64 + 8 * st.stage, st.phase ^ 1u);
            if (kb == 0 && st.rank == 0 && probe_i < 8) MM_PROBE(probe_i, 5);
            const uint32_t full = st.bars + 8 * st.stage;
            const uint32_t sa = st.base + st.stage * kStageBytes, sb = sa + BM * BK * 2;
            if (st.rank == 0) mbar_expect_tx(full, tx);
            const uint32_t full_lead = map_rank(full, 0u);
            tma_load_2d_pair(sa, &P.ta, full_lead, kb * BK, arow);
            tma_load_2d_pair(sb, tmb, full_lead, kb * BK, brow);
            if (++st.stage == S) { st.stage = 0; st.phase ^= 1u; }
        }
    }
    template <class F>
    __device__ static void run(const Params& P, State& st, char*, F& f, const KlLaunch* L) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int nk = P.K / BK;
        if (warp == 0 && lane == 0 && st.rank == 0) {
            // scheduler (the leader's thread 0, which owns the launcher's fetch state): the first
            // tile at once, each next one when the leader's producer asks; publishing needs a
            // cluster-scope release, which this thread -- unlike the producer with its TMA loads
            // in flight -- pays without waiting
            for (uint32_t i = 0;; ++i) {
                if (i >= 1) mbar_wait(st.bars + 200, (i - 1u) & 1u);
                const uint32_t item = f.next();
                const uint32_t q = i % kTileQ;
                if (i >= kTileQ) mbar_wait_cl(st.bars + 256 + 8 * q, (i / kTileQ - 1u) & 1u);
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(st.bars + 320 + 4 * q), "r"(item) : "memory");
                st_cluster_u32(map_rank(st.bars + 320 + 4 * q, 1u), item);
                mbar_arrive_local(st.bars + 160 + 8 * q);
                mbar_arrive_cl(map_rank(st.bars + 160 + 8 * q, 1u));
                if (i < 8) MM_PROBE(i, 4);
                if (item == kItemNone) break;
            }
        } else if (warp == 2 && lane == 0) {
            for (uint32_t i = 0;; ++i) {                     // producers (both CTAs)
                const uint32_t item = tile_item(st, i);
                tile_release(st, i);
                if (item == kItemNone) break;
                load_tile(P, st, item, i);
            }
        } else if (warp == 1 && lane == 0 && st.rank == 0) {
            tc_fence_after();
            for (uint32_t i = 0;; ++i) {                     // MMA issuer
                const uint32_t item = tile_item(st, i);
                if (i < 8) MM_PROBE(i, 6);
                tile_release(st, i);
                if (item == kItemNone) break;
                const uint32_t acc = i & 1u, u = i >> 1;
                if (u >= 1) mbar_wait_cl(st.bars + 144 + 8 * acc, (u - 1u) & 1u);
                if (i < 8) MM_PROBE(i, 7);
                tc_fence_after();
                const uint32_t idesc = (item & 3u) ? kIdescHalf : kIdesc;
                const uint32_t tacc = st.tmem + acc * BN;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(st.bars + 8 * st.stage, st.phase);
                    tc_fence_after();
                    if (kb == 0 && i < 8) MM_PROBE(i, 0);
                    const uint32_t sa = st.base + st.stage * kStageBytes, sb = sa + BM * BK * 2;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        umma_bf16_pair(tacc, umma_desc(sa + k * 32), umma_desc(sb + k * 32), idesc,
                                       (kb | k) != 0 ? 1u : 0u);
                    umma_commit_pair(st.bars + 64 + 8 * st.stage);
                    if (++st.stage == S) { st.stage = 0; st.phase ^= 1u; }
                }
                umma_commit_pair(st.bars + 128 + 8 * acc);
                if (i < 8) MM_PROBE(i, 1);
            }
        } else if (warp >= 4) {
            const int tiles_n = P.N / BN;
            for (uint32_t i = 0;; ++i) {                     // epilogue warps
                const uint32_t item = tile_item(st, i);
                __syncwarp();
                if (lane == 0) tile_release(st, i);
                if (item == kItemNone) break;
                const uint32_t vb = item >> 2;
                const int part = (int)(item & 3u);
                const int tm = (int)vb / tiles_n, tn = (int)vb % tiles_n;
                const uint32_t acc = i & 1u;
                drain_tile(P, st, tm, tn * BN + (part == 2 ? BN / 2 : 0), part ? BN / 2 : BN, acc, (i >> 1) & 1u, i);
                __syncwarp();
                if (lane == 0) {
                    if (st.rank == 0) mbar_arrive_local(st.bars + 144 + 8 * acc);
                    else mbar_arrive_cl(map_rank(st.bars + 144 + 8 * acc, 0u));
                    if (warp == 4 && st.rank == 0) {
                        if (i < 8) MM_PROBE(i, 3);
                        if (L && L->audit) atomicAdd(L->audit + vb, 1u);
                        if (L && L->stamps) L->stamps[2 * (size_t)vb + 1] = gtimer();
                    }
                }
            }
        }
        __syncwarp();
    }
    __device__ static void block(const Params& P, State& st, char* d, uint32_t vb) { block_part(P, st, d, vb, 0); }
    // part 0: the whole 256x256 tile vb; part 1 / 2: its left / right 256x128 half (the plain
    // grid splits its last, partial round of tiles so every pair gets work: wave quantisation).
    // Every output element is the same k-ordered tensor-core accumulation either way.
    __device__ static void block_part(const Params& P, State& st, char*, uint32_t vb, int part) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int tiles_n = P.N / BN;
        const int tm = (int)vb / tiles_n, tn = (int)vb % tiles_n;
        const int nk = P.K / BK;
        const int w = part ? BN / 2 : BN;                     // tile width (columns)
        const int col = tn * BN + (part == 2 ? BN / 2 : 0);   // first column
        const CUtensorMap* tmb = part ? &P.tbh : &P.tb;
        const uint32_t idesc = part ? kIdescHalf : kIdesc;
        const uint32_t tx = 2u * (uint32_t)(BM * BK * 2 + (w / 2) * BK * 2);   // both CTAs' bytes
        const uint32_t acc = st.ntile & 1u;                 // accumulator of this tile
        if (warp == 0) {
            if (lane == 0) {
                uint32_t s = st.stage, ph = st.phase;
                const int arow = tm * (2 * BM) + (int)st.rank * BM, brow = col + (int)st.rank * (w / 2);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(st.bars + 64 + 8 * s, ph ^ 1u);
                    const uint32_t full = st.bars + 8 * s;
                    const uint32_t sa = st.base + s * kStageBytes, sb = sa + BM * BK * 2;
#ifdef KL_MM_DBG_NOTMA   // A/B probe: the MMAs on stale shared memory, no operand traffic
                    if (st.rank == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(full) : "memory");
                    (void)sa; (void)sb; (void)arow; (void)brow; (void)tmb; (void)tx;
#else
                    if (st.rank == 0) mbar_expect_tx(full, tx);
                    const uint32_t full_lead = map_rank(full, 0u);
                    tma_load_2d_pair(sa, &P.ta, full_lead, kb * BK, arow);
                    tma_load_2d_pair(sb, tmb, full_lead, kb * BK, brow);
#endif
                    if (++s == S) { s = 0; ph ^= 1u; }
                }
            }
            __syncwarp();
        } else if (warp == 1) {
            if (st.rank == 0) {
                tc_fence_after();
                if (lane == 0) {
                    uint32_t s = st.stage, ph = st.phase;
                    const uint32_t tacc = st.tmem + acc * BN;
                    for (int kb = 0; kb < nk; ++kb) {
                        mbar_wait(st.bars + 8 * s, ph);
                        tc_fence_after();
                        if (kb == 0) MM_PROBE(st.ntile, 0);
                        const uint32_t sa = st.base + s * kStageBytes, sb = sa + BM * BK * 2;
#ifndef KL_MM_DBG_NOMMA   // A/B probe: operand traffic only
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k)
                            umma_bf16_pair(tacc, umma_desc(sa + k * 32), umma_desc(sb + k * 32), idesc,
                                           (kb | k) != 0 ? 1u : 0u);
#else
                        (void)sa; (void)sb; (void)tacc; (void)idesc;
#endif
                        umma_commit_pair(st.bars + 64 + 8 * s);   // stage free in both CTAs
                        if (++s == S) { s = 0; ph ^= 1u; }
                    }
                    umma_commit_pair(st.bars + 128 + 8 * acc);    // accumulator `acc` complete
                    MM_PROBE(st.ntile, 1);
                }
                __syncwarp();
            }
        } else if (warp >= 4 && st.prev_m >= 0) {
            drain(P, st, st.prev_m, st.prev_col, st.prev_w, acc ^ 1u);   // previous tile, other accumulator
        }
        // every role advances the shared pipeline state identically
        for (int kb = 0; kb < nk; ++kb)
            if (++st.stage == S) { st.stage = 0; st.phase ^= 1u; }
        if (st.prev_m >= 0) st.tph ^= 1u << (acc ^ 1u);    // that accumulator's wait was consumed
        st.prev_m = tm;
        st.prev_col = col;
        st.prev_w = w;
        st.ntile++;
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }
};

}  // namespace

namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

bool encode_kmajor(CUtensorMap* m, const void* base, uint64_t rows, uint64_t k, int box_rows) {
    auto fn = get_encode();
    if (!fn) return false;
    cuuint64_t dims[2] = {k, rows};
    cuuint64_t strides[1] = {k * 2};
    cuuint32_t box[2] = {BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// C [rows][cols] fp32, box 32 x 32, 128B swizzle (the epilogue's staging layout).
bool encode_c(CUtensorMap* m, void* base, uint64_t rows, uint64_t cols) {
    auto fn = get_encode();
    if (!fn) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 4};
    cuuint32_t box[2] = {(cuuint32_t)kEpiBox, (cuuint32_t)kEpiBox};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Stage count of a launch: L.variant names it (0 = the default, the deepest ring).
int stages_of(uint32_t variant) {
    for (int v : kStageLevels)
        if ((int)variant == v) return v;
    return 6;
}

}  // namespace

#ifdef KL_MM_PROBE
extern "C" int kl_mm_probe_read(unsigned long long* out, int n) {
    const int cap = 96 * kProbeStride;
    if (n > cap) n = cap;
    cudaError_t e = cudaMemcpyFromSymbol(out, g_mm_probe, sizeof(unsigned long long) * n);
    static unsigned long long zero[96 * kProbeStride];
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_mm_probe, zero, sizeof zero);
    return (int)e;
}
extern "C" int kl_mm_probe_stride() { return kProbeStride; }
#endif

int kl_mm_stage_smem(int stages) {     // dynamic shared memory of one CTA at `stages`
    return stages * kStageBytes + kEpiBytes + 1024 + kBarBytes;
}

int kl_mm_info(KlKindInfo* o) {
    if (!get_encode()) return -3;
    int rc = 0;
    KlKindInfo tmp;
    // every instantiation's attributes are set (dynamic shared memory opt-in) at load time
    if ((rc = info_of_pair<BodyMM<2>>(&tmp)) || (rc = info_of_pair<BodyMM<3>>(&tmp)) ||
        (rc = info_of_pair<BodyMM<4>>(&tmp)))
        return rc;
    rc = info_of_pair<BodyMM<6>>(o);
    if (rc) return rc;
    o->tmem_cols = (int)kTmemCols;
    o->dyn_smem = kl_mm_stage_smem(2);   // the kind's profile: its shallowest ring (the runtime
                                         // picks each launch's depth, kl_runtime.cpp variant_of)
    return 0;
}

int kl_mm_prepare(const void* args, uint32_t bytes, uint32_t grid, void* blob, uint32_t cap) {
    if (bytes != sizeof(kl_args_mm) || cap < sizeof(MMParams)) return -1;
    const kl_args_mm& a = *reinterpret_cast<const kl_args_mm*>(args);
    if (a.M <= 0 || a.N <= 0 || a.K <= 0 || a.M % (2 * BM) || a.N % BN || a.K % BK) return -1;
    if ((uint64_t)grid > (uint64_t)(a.M / (2 * BM)) * (uint64_t)(a.N / BN)) return -1;   // one tile per block
    MMParams p;
    std::memset(&p, 0, sizeof p);
    if (!encode_kmajor(&p.ta, a.A, (uint64_t)a.M, (uint64_t)a.K, BM)) return -1;
    if (!encode_kmajor(&p.tb, a.Bt, (uint64_t)a.N, (uint64_t)a.K, BNH)) return -1;
    if (!encode_kmajor(&p.tbh, a.Bt, (uint64_t)a.N, (uint64_t)a.K, BNH / 2)) return -1;
    if (!encode_c(&p.tc, a.C, (uint64_t)a.M, (uint64_t)a.N)) return -1;
    p.C = a.C;
    p.M = a.M;
    p.N = a.N;
    p.K = a.K;
    std::memcpy(blob, &p, sizeof p);
    return 0;
}

int kl_mm_launch_persistent(const void* blob, const KlLaunch& L, uint32_t grid, void* stream) {
    // a short remainder (uncapped launch sized to the remaining tiles) still gets two CTAs per tile
    if (grid < L.n_sms) grid = std::min(2u * grid, L.n_sms);
    switch (stages_of(L.variant)) {
        case 2: return launch_persistent_pair<BodyMM<2>>(blob, L, grid, stream);
        case 3: return launch_persistent_pair<BodyMM<3>>(blob, L, grid, stream);
        case 4: return launch_persistent_pair<BodyMM<4>>(blob, L, grid, stream);
        default: return launch_persistent_pair<BodyMM<6>>(blob, L, grid, stream);
    }
}

int kl_mm_launch_plain(const void* blob, uint32_t offset, uint32_t n, void* stream) {
    return launch_plain_pair<BodyMM<6>>(blob, offset, n, stream);
}
