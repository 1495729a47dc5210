// kl_mm.cu -- MM ("Multiplying two dense matrices", 8192x2048 . 2048x2048) on the
// 5th-generation tensor cores (product path).
//
// One virtual thread block = one 128x256 fp32 output tile.  A persistent block (8 warps) pulls
// tiles from the slice launcher and runs, per tile,
//   warp 0 lane 0 : TMA producer  -- 128x64 (A) and 256x64 (B) bf16 tiles, 128B swizzle, into a
//                   ring of kStages shared-memory stages, completion on mbarriers (expect_tx);
//   warp 1 lane 0 : MMA issuer    -- tcgen05.mma.cta_group::1.kind::f16 (M=128, N=256, K=16) x4
//                   per stage into one of two 256-column fp32 TMEM accumulators; tcgen05.commit
//                   frees the stage; the last commit signals the epilogue;
//   warps 4..7    : epilogue      -- drains the PREVIOUS tile's accumulator (tcgen05.ld
//                   32x32b.x32, each warp its 32 TMEM lanes) while warps 0-1 run this tile's
//                   mainloop; the last tile is drained in fini().  Warps 2-3 idle (8 warps keep
//                   b*wpb divisible by the 4 schedulers: whole virtual-SM warps, R14).
// The stage count is the kernel's occupancy knob (shared memory per block).
// Numerics: bf16 products are exact in fp32; only the fp32 accumulation order differs from the
// oracle's fp64 sum (normwise tolerance).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstring>
#include "kl_internal.h"
#include "kl_launcher.cuh"

namespace {

constexpr int BM = 128, BN = 256, BK = 64;
#ifndef KL_MM_STAGES
#define KL_MM_STAGES 4   // the stage count is a build knob: 2-4 (48 KiB of shared memory each)
#endif
constexpr int kStages = KL_MM_STAGES;
static_assert(kStages >= 2 && kStages <= 4, "KL_MM_STAGES in [2, 4] (227 KB of shared memory per block)");
constexpr int kStageBytes = (BM + BN) * BK * 2;          // 48 KiB
constexpr int kBarOffset = kStages * kStageBytes;
constexpr int kDynSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
constexpr int kThreads = 256;   // 8 warps: whole warps per virtual SM (R14)
constexpr uint32_t kTmemCols = 2 * BN;   // two fp32 accumulators: tile i's MMAs overlap tile i-1's epilogue
// instruction descriptor: F32 accumulate, BF16 A/B, K-major A/B, N = 256, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

struct MMParams {
    CUtensorMap ta;   // A  [M][K] bf16, box 64 x 128
    CUtensorMap tb;   // Bt [N][K] bf16, box 64 x 256
    float* C;
    int32_t M, N, K;
};
static_assert(sizeof(MMParams) <= 512, "blob");

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

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
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"((uint64_t)map), "r"(bar), "r"(c0), "r"(c1)
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
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
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

struct BodyMM {
    using Params = MMParams;
    static constexpr int kThreads = ::kThreads, kChunk = 1, kDynSmem = ::kDynSmem;
    struct State {
        uint32_t base;      // 1024-aligned shared address of stage 0
        uint32_t bars;      // full[s] bars+8s, empty[s] bars+64+8s, tfull[b] bars+128+8b, tmem ptr bars+192
        uint32_t tmem;
        uint32_t stage, phase;
        uint32_t tph;       // per-accumulator wait parity bits
        uint32_t ntile;     // tiles issued by this persistent block
        int prev_m, prev_n; // tile whose accumulator is still to be drained (-1: none)
    };
    __device__ static void init(const Params&, State& st, char* dsmem) {
        const uint32_t raw = smem_u32(dsmem);
        st.base = (raw + 1023u) & ~1023u;
        st.bars = st.base + kBarOffset;
        st.stage = st.phase = st.tph = st.ntile = 0;
        st.prev_m = st.prev_n = -1;
        const int warp = threadIdx.x >> 5;
        if (threadIdx.x == 0) {
            for (int s = 0; s < kStages; ++s) {
                mbar_init(st.bars + 8 * s, 1);
                mbar_init(st.bars + 64 + 8 * s, 1);
            }
            mbar_init(st.bars + 128, 1);
            mbar_init(st.bars + 136, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        if (warp == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(st.bars + 192),
                         "r"(kTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(st.tmem) : "r"(st.bars + 192));
    }
    // Epilogue warps: wait for tile (m, n)'s accumulator b, move it TMEM -> registers -> C.
    __device__ static void drain(const Params& P, State& st, int m, int n, uint32_t b) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        mbar_wait(st.bars + 128 + 8 * b, (st.tph >> b) & 1u);
        tc_fence_after();
        const int q = warp & 3;                              // TMEM lane quarter of this warp
        const int row = m * BM + q * 32 + lane;
        float* crow = P.C + (size_t)row * P.N + (size_t)n * BN;
        const uint32_t tbase = st.tmem + ((uint32_t)(q * 32) << 16) + b * BN;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
            uint32_t r[32];
            TMEM_LD_X32(tbase + (uint32_t)c, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            float4* dst = reinterpret_cast<float4*>(crow + c);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                dst[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                     __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
        }
        tc_fence_before();
    }
    __device__ static void fini(const Params& P, State& st, char*) {
        if (st.prev_m >= 0 && (threadIdx.x >> 5) >= 4) drain(P, st, st.prev_m, st.prev_n, (st.ntile - 1) & 1u);
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        if ((threadIdx.x >> 5) == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(st.tmem), "r"(kTmemCols));
    }
    __device__ static void block(const Params& P, State& st, char*, uint32_t vb) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int tiles_n = P.N / BN;
        const int tm = (int)vb / tiles_n, tn = (int)vb % tiles_n;
        const int nk = P.K / BK;
        const uint32_t acc = st.ntile & 1u;                 // accumulator of this tile
        if (warp == 0) {
            if (lane == 0) {
                uint32_t s = st.stage, ph = st.phase;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(st.bars + 64 + 8 * s, ph ^ 1u);
                    const uint32_t full = st.bars + 8 * s;
                    const uint32_t sa = st.base + s * kStageBytes, sb = sa + BM * BK * 2;
                    mbar_expect_tx(full, kStageBytes);
                    tma_load_2d(sa, &P.ta, full, kb * BK, tm * BM);
                    tma_load_2d(sb, &P.tb, full, kb * BK, tn * BN);
                    if (++s == kStages) { s = 0; ph ^= 1u; }
                }
            }
            __syncwarp();
        } else if (warp == 1) {
            tc_fence_after();
            if (lane == 0) {
                uint32_t s = st.stage, ph = st.phase;
                const uint32_t tacc = st.tmem + acc * BN;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(st.bars + 8 * s, ph);
                    tc_fence_after();
                    const uint32_t sa = st.base + s * kStageBytes, sb = sa + BM * BK * 2;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        umma_bf16(tacc, umma_desc(sa + k * 32), umma_desc(sb + k * 32), kIdesc,
                                  (kb | k) != 0 ? 1u : 0u);
                    umma_commit(st.bars + 64 + 8 * s);       // stage free once these MMAs finish
                    if (++s == kStages) { s = 0; ph ^= 1u; }
                }
                umma_commit(st.bars + 128 + 8 * acc);        // accumulator `acc` complete
            }
            __syncwarp();
        } else if (warp >= 4 && st.prev_m >= 0) {
            drain(P, st, st.prev_m, st.prev_n, acc ^ 1u);    // previous tile, other accumulator
        }
        // every role advances the shared pipeline state identically
        for (int kb = 0; kb < nk; ++kb)
            if (++st.stage == kStages) { st.stage = 0; st.phase ^= 1u; }
        if (st.prev_m >= 0) st.tph ^= 1u << (acc ^ 1u);    // that accumulator's wait was consumed
        st.prev_m = tm;
        st.prev_n = tn;
        st.ntile++;
        tc_fence_before();
        __syncthreads();   // the drained accumulator is free before the next tile's first MMA
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

}  // namespace

int kl_mm_info(KlKindInfo* o) {
    if (!get_encode()) return -3;
    int rc = info_of<BodyMM>(o);
    if (rc) return rc;
    o->tmem_cols = (int)kTmemCols;
    return 0;
}

int kl_mm_prepare(const void* args, uint32_t bytes, uint32_t grid, void* blob, uint32_t cap) {
    if (bytes != sizeof(kl_args_mm) || cap < sizeof(MMParams)) return -1;
    const kl_args_mm& a = *reinterpret_cast<const kl_args_mm*>(args);
    if (a.M <= 0 || a.N <= 0 || a.K <= 0 || a.M % BM || a.N % BN || a.K % BK) return -1;
    if ((uint64_t)grid > (uint64_t)(a.M / BM) * (uint64_t)(a.N / BN)) return -1;   // one tile per block
    MMParams p;
    std::memset(&p, 0, sizeof p);
    if (!encode_kmajor(&p.ta, a.A, (uint64_t)a.M, (uint64_t)a.K, BM)) return -1;
    if (!encode_kmajor(&p.tb, a.Bt, (uint64_t)a.N, (uint64_t)a.K, BN)) return -1;
    p.C = a.C;
    p.M = a.M;
    p.N = a.N;
    p.K = a.K;
    std::memcpy(blob, &p, sizeof p);
    return 0;
}

int kl_mm_launch_persistent(const void* blob, const KlLaunch& L, uint32_t grid, void* stream) {
    return launch_persistent<BodyMM>(blob, L, grid, stream);
}

int kl_mm_launch_plain(const void* blob, uint32_t offset, uint32_t n, void* stream) {
    return launch_plain<BodyMM>(blob, offset, n, stream);
}
