// kl_kernels.cu -- sm_100a slice launcher and the paper's benchmark kernels (product path).
//
// Slicing: a slice is a contiguous range of a kernel's thread blocks launched with
// its block index rectified by an offset.  On B200 a phase launches ONE persistent grid per
// kernel (cap x n_SM blocks); each admitted block pulls virtual block ids from the kernel's
// slice control word and runs Body::block(vb) -- index rectification as a kernel parameter
// instead of Fermi SASS rewriting.  Occupancy control (P:258-267 via slice sizes on
// Fermi) becomes a per-SM admission cap read from %smid.
//
// Every body computes exactly the definition in oracle/kernels.c (independently written); the
// per-output operation order never depends on the slicing, so sliced == unsliced bit for bit.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstring>
#include "kl_internal.h"
#include "kl_launcher.cuh"

namespace {

// ------------------------------------------------------------------------------------------
// Benchmark bodies.  Interface: Params (kernel args), kThreads, kChunk (default virtual blocks
// per fetch), State + init/fini (per persistent block), block(vb) (one virtual thread block).
// ------------------------------------------------------------------------------------------
struct Empty {};

// PC: 256 threads; dependent loads through the read-only path.
#ifndef KL_MINB_ST
#define KL_MINB_ST 16
#endif
#ifndef KL_MINB_MRIQ
#define KL_MINB_MRIQ 8
#endif
#ifndef KL_MINB_BS
#define KL_MINB_BS 9
#endif
struct BodyPC {
    using Params = kl_args_pc;
    using State = Empty;
    static constexpr int kThreads = 256, kChunk = 1, kDynSmem = 0, kMinBlocks = 8;
    __device__ static void init(const Params&, State&, char*) {}
    __device__ static void fini(const Params&, State&, char*) {}
    __device__ static void block(const Params& a, State&, char*, uint32_t vb) {
        uint32_t t = vb * 256u + threadIdx.x;
        if (t >= a.n_threads) return;
        uint32_t p = (t * 2654435761u) % a.n_nodes;
        uint32_t acc = 0;
        for (uint32_t h = 0; h < a.hops; ++h) {
            p = (uint32_t)__ldg(a.next + p);
            acc += p;
        }
        a.out[t] = (int32_t)p;
        a.acc[t] = acc;
    }
};

// SAD: one warp per 16x16 macroblock; the 48x48 clamped reference window is staged in
// shared memory, the current block lives in registers; lane l owns displacement column dx = l
// and sweeps all 33 dy with vabsdiff4 (4 pixels per instruction); column dx = 32 is spread over
// the lanes afterwards.
__device__ __forceinline__ uint32_t vsad4(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
struct BodySAD {
    using Params = kl_args_sad;
    using State = Empty;
    // 32 one-warp blocks per SM (the block limit) at <= 64 registers.  The round-1 body kept the
    // whole 16x16 current macroblock (64 words) and 33 accumulators in registers: 128 registers,
    // 16 resident warps, too few to cover the window loads (ncu: alu pipe 53 %, long-scoreboard
    // stalls).  Here each of two passes holds half the macroblock's rows (32 words) and a ring of
    // 8 accumulators; pass 0 parks its partial sums in shared memory, pass 1 adds them.
    // Four warps per block, each on its own macroblock: a fetched chunk of 4 virtual blocks runs
    // together (block_range), so the launcher's per-block join / fetch / leave atomics are paid
    // once per 4 macroblocks (with one-warp blocks they cost +50 % against the plain grid).
    static constexpr int kThreads = 128, kChunk = 4, kDynSmem = 0, kMinBlocks = 8;
    __device__ static void init(const Params&, State&, char*) {}
    __device__ static void fini(const Params&, State&, char*) {}
    // One pass over macroblock rows r in [8H, 8H + 8) (cur: their 32 words).  Lane l =
    // displacement column dx = l; SAD(dx, dy) gets the row term S(y, r) of window row y = dy + r.
    // Window row y feeds dy = y - r for the pass's 8 rows, so 8 accumulators in a ring indexed by
    // dy mod 8 suffice; the one for dy = y - (8H + 7) is complete after row y.  The 40 window rows
    // come in 5 phases of 8 (only the first and last phase have invalid (y, r) pairs), so every
    // ring index and validity test is a compile-time constant.
    template <int H, int P>
    __device__ static void phase(const uint32_t* win, const uint32_t (&cur)[32], int lane, uint32_t (&ring)[8],
                                 uint16_t* part, uint16_t* o) {
        const int wo = lane >> 2, sh = (lane & 3) * 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int y = 8 * H + 8 * P + j;
            const uint32_t* row = win + y * 12 + wo;
            const uint32_t w0 = row[0], w1 = row[1], w2 = row[2], w3 = row[3], w4 = row[4];
            const uint32_t q0 = __funnelshift_r(w0, w1, sh), q1 = __funnelshift_r(w1, w2, sh);
            const uint32_t q2 = __funnelshift_r(w2, w3, sh), q3 = __funnelshift_r(w3, w4, sh);
#pragma unroll
            for (int rr = 0; rr < 8; ++rr) {
                const bool valid = (P == 0) ? (rr <= j) : (P == 4) ? (rr >= j) : true;   // 0 <= dy <= 32
                if (valid) {
                    uint32_t& acc = ring[(j - rr + 8) & 7];
                    uint32_t s = vsad4(q0, cur[rr * 4 + 0], acc);
                    s = vsad4(q1, cur[rr * 4 + 1], s);
                    s = vsad4(q2, cur[rr * 4 + 2], s);
                    acc = vsad4(q3, cur[rr * 4 + 3], s);
                }
            }
            const int dy = 8 * P + j - 7;                  // complete: all 8 rows of the pass added
            if (dy >= 0) {
                uint32_t& acc = ring[(j + 1) & 7];         // dy mod 8
                if (H == 0) part[dy * 32 + lane] = (uint16_t)acc;                 // <= 8*16*255
                else o[dy * 33 + lane] = (uint16_t)(acc + part[dy * 32 + lane]);  // <= 65280
                acc = 0;
            }
        }
    }
    template <int H>
    __device__ static uint32_t half(const uint32_t* win, const uint32_t* curw, int lane, uint16_t* part, uint16_t* o,
                                    uint32_t col) {
        uint32_t cur[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) cur[i] = curw[H * 32 + i];
        uint32_t ring[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) ring[i] = 0;
        phase<H, 0>(win, cur, lane, ring, part, o);
        phase<H, 1>(win, cur, lane, ring, part, o);
        phase<H, 2>(win, cur, lane, ring, part, o);
        phase<H, 3>(win, cur, lane, ring, part, o);
        phase<H, 4>(win, cur, lane, ring, part, o);
        // displacement column dx = 32 (lane l: dy = l; lane 0 also dy = 32 in the high half)
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
            const uint32_t* row = win + (lane + 8 * H + rr) * 12 + 8;
#pragma unroll
            for (int i = 0; i < 4; ++i) col = vsad4(row[i], cur[rr * 4 + i], col);
        }
        return col;
    }
    __device__ static void block_range(const Params& a, State& st, char* d, uint32_t v0, uint32_t v1) {
        const uint32_t v = v0 + (threadIdx.x >> 5);
        if (v < v1) macroblock(a, v);
    }
    // One warp: macroblock vb (its own slice of the block's shared memory).
    __device__ static void macroblock(const Params& a, uint32_t vb) {
        __shared__ uint32_t win_all[4][48 * 12];
        __shared__ uint32_t curw_all[4][64];
        __shared__ uint16_t part_all[4][33 * 32];
        const int wid = threadIdx.x >> 5;
        uint32_t* win = win_all[wid];
        uint32_t* curw = curw_all[wid];
        uint16_t* part = part_all[wid];
        const int W = a.width, H = a.height, mbw = W / 16, n_mb = mbw * (H / 16);
        if ((int)vb >= n_mb) return;   // padding blocks of the paper's 8048-block grid
        const int lane = threadIdx.x & 31;
        const int mx = vb % mbw, my = vb / mbw;
        const int x0 = mx * 16 - 16, y0 = my * 16 - 16;
        const bool inner = (x0 >= 0) && (x0 + 48 <= W) && (y0 >= 0) && (y0 + 48 <= H);
        for (int i = lane; i < 48 * 12; i += 32) {
            int y = i / 12, wc = i % 12;
            if (inner) {
                win[i] = *reinterpret_cast<const uint32_t*>(a.ref + (size_t)(y0 + y) * W + x0 + wc * 4);
            } else {
                int gy = min(max(y0 + y, 0), H - 1);
                uint32_t v = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    int gx = min(max(x0 + wc * 4 + b, 0), W - 1);
                    v |= (uint32_t)a.ref[(size_t)gy * W + gx] << (8 * b);
                }
                win[i] = v;
            }
        }
        for (int i = lane; i < 64; i += 32)
            curw[i] = *reinterpret_cast<const uint32_t*>(a.cur + (size_t)(my * 16 + i / 4) * W + mx * 16 + (i % 4) * 4);
        __syncwarp();
        uint16_t* o = a.out + (size_t)vb * 1089;
        uint32_t col = half<0>(win, curw, lane, part, o, 0u);
        __syncwarp();
        col = half<1>(win, curw, lane, part, o, col);
        o[lane * 33 + 32] = (uint16_t)col;
        if (lane == 0) {               // dy = 32 of column dx = 32
            uint32_t s = 0;
#pragma unroll 4
            for (int r = 0; r < 16; ++r)
#pragma unroll
                for (int i = 0; i < 4; ++i) s = vsad4(win[(32 + r) * 12 + 8 + i], curw[r * 4 + i], s);
            o[32 * 33 + 32] = (uint16_t)s;
        }
        __syncwarp();
    }
};

// SPMV (CUSP CSR-vector): 8 rows per virtual block, the paper's unit of work.  At this
// size the kernel is latency-bound (row pointer -> column -> x gather -> reduce per row), so rows
// in flight is what counts.  A block runs a whole fetched chunk of 8 virtual blocks (64 rows)
// together, 4 lanes per row (rows hold 8-24 nonzeros: 2-6 per lane), lane-strided products and a
// butterfly inside the row's lane group -- 8x the rows in flight of a warp per row, with the same
// number of blocks, joins and fetches (round 1: more, smaller blocks lost their gain to the
// launcher's per-block costs).  A row's arithmetic never depends on the grouping.
struct BodySPMV {
    using Params = kl_args_spmv;
    using State = Empty;
    static constexpr int kLanes = 4;
    static constexpr int kThreads = 256, kChunk = 8, kDynSmem = 0, kMinBlocks = 8;
    __device__ static void init(const Params&, State&, char*) {}
    __device__ static void fini(const Params&, State&, char*) {}
    __device__ static void block_range(const Params& a, State&, char*, uint32_t v0, uint32_t v1) {
        const int r_local = (int)(threadIdx.x / kLanes), lane = (int)(threadIdx.x % kLanes);
        const int row = (int)v0 * 8 + r_local;
        const bool live = r_local < (int)(v1 - v0) * 8 && row < a.n_rows;   // the warp takes the shuffles
        const int s = live ? __ldg(a.rowptr + row) : 0, e = live ? __ldg(a.rowptr + row + 1) : 0;
        float sum = 0.f;
        // batches of kB products per lane: all kB (column, value) loads in flight together, then
        // all kB x gathers, then the fmaf chain in j order (the same order as a plain loop over
        // j = s + lane, s + lane + kLanes, ...): two dependent memory round trips per batch instead
        // of two per product (rows of <= kB * kLanes = 24 nonzeros take one batch)
        constexpr int kB = 6;
        for (int j0 = s + lane; j0 < e; j0 += kB * kLanes) {
            int c[kB];
            float v[kB], xv[kB];
#pragma unroll
            for (int b = 0; b < kB; ++b) {
                const int j = j0 + b * kLanes;
                c[b] = j < e ? __ldg(a.cols + j) : 0;
                v[b] = j < e ? __ldg(a.vals + j) : 0.f;
            }
#pragma unroll
            for (int b = 0; b < kB; ++b) xv[b] = (j0 + b * kLanes < e) ? __ldg(a.x + c[b]) : 0.f;
#pragma unroll
            for (int b = 0; b < kB; ++b)
                if (j0 + b * kLanes < e) sum = fmaf(v[b], xv[b], sum);
        }
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        if (live && lane == 0) a.y[row] = sum;
    }
};

// ST (Parboil 7-point stencil): 32x4 (x,y) tile, 64 z-points per block; the z
// neighbours ride a register queue, x/y neighbours come through L1.
struct BodyST {
    // Tile 128 (x) x 4 (y) x 32 (z) per block: each thread owns 4 consecutive x (one float4) of
    // one row and marches z with a register queue (z-1, z, z+1); x neighbours come from the
    // adjacent lanes by shuffle (lanes 0 / 31 load the tile-edge column), y neighbours are float4
    // loads through L1.  ~11 instructions per point instead of ~40 with one point per thread, so
    // the kernel is no longer issue-bound.  Interior points: the same operand order and fmaf as
    // the oracle's definition (bit-identical); boundary points copy the input.  nx % 4 == 0.
    using Params = kl_args_st;
    using State = Empty;
    static constexpr int kThreads = 128, kChunk = 1, kDynSmem = 0, kMinBlocks = KL_MINB_ST;
    __device__ static void init(const Params&, State&, char*) {}
    __device__ static void fini(const Params&, State&, char*) {}
    static constexpr int kTz = 32;   // z points per block (kl_inputs.ST_TILE)
    __device__ static float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
    __device__ static void block(const Params& a, State&, char*, uint32_t vb) {
        const int nx = a.nx, ny = a.ny, nz = a.nz;
        const int gx = (nx + 127) / 128, gy = (ny + 3) / 4;
        const int bx = vb % gx, by = (vb / gx) % gy, bz = vb / (gx * gy);
        const int lane = threadIdx.x & 31;
        const int x0 = bx * 128 + lane * 4, y = by * 4 + (threadIdx.x >> 5);
        if (y >= ny) return;                      // whole warp (one row per warp)
        const bool act = x0 < nx;
        const int z0 = bz * kTz, z1 = min(z0 + kTz, nz);
        if (z0 >= nz) return;                     // a grid larger than the field: nothing to do
        const size_t sz = (size_t)nx * ny;
        const bool iy = y > 0 && y < ny - 1;
        const float* in = a.in;
        size_t f = (size_t)z0 * sz + (size_t)y * nx + (act ? x0 : 0);
        const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
        float4 zm = (act && z0 > 0) ? ld4(in + f - sz) : zero;
        float4 c = act ? ld4(in + f) : zero;
        for (int z = z0; z < z1; ++z, f += sz) {
            const float4 zp = (act && z + 1 < nz) ? ld4(in + f + sz) : zero;
            const bool inner = iy && z > 0 && z < nz - 1;
            // x neighbours of the float4: lane-1's .w and lane+1's .x (same row, same z)
            float xm = __shfl_up_sync(0xffffffffu, c.w, 1);
            float xp = __shfl_down_sync(0xffffffffu, c.x, 1);
            if (act && inner) {
                if (lane == 0 && x0 > 0) xm = __ldg(in + f - 1);
                if ((lane == 31 || x0 + 4 >= nx) && x0 + 4 < nx) xp = __ldg(in + f + 4);
                const float4 ym = ld4(in + f - nx), yp = ld4(in + f + nx);
#ifdef KL_ST_X2
                // FP32x2 path (measured, not the default): elements (0, 1) and (2, 3) in pairs --
                // FADD2 / FMUL2 / FFMA2 round each lane exactly like the scalar fadd / fmul / fmaf
                // below, same operand order (bit-identical); 14 instead of 28 FP instructions per
                // float4.  Plain grid 0.190 -> 0.186 ms, but the persistent variant 0.213 -> 0.241
                // ms solo and C5 within noise (+0.6 %), so the scalar body stays the default.
                float2 s0 = __fadd2_rn(make_float2(zm.x, zm.y), make_float2(zp.x, zp.y));
                float2 s1 = __fadd2_rn(make_float2(zm.z, zm.w), make_float2(zp.z, zp.w));
                s0 = __fadd2_rn(s0, make_float2(ym.x, ym.y));
                s1 = __fadd2_rn(s1, make_float2(ym.z, ym.w));
                s0 = __fadd2_rn(s0, make_float2(yp.x, yp.y));
                s1 = __fadd2_rn(s1, make_float2(yp.z, yp.w));
                s0 = __fadd2_rn(s0, make_float2(xm, c.x));
                s1 = __fadd2_rn(s1, make_float2(c.y, c.z));
                s0 = __fadd2_rn(s0, make_float2(c.y, c.z));
                s1 = __fadd2_rn(s1, make_float2(c.w, xp));
                const float2 n0 = __fmul2_rn(make_float2(a.c0, a.c0), make_float2(c.x, c.y));
                const float2 n1 = __fmul2_rn(make_float2(a.c0, a.c0), make_float2(c.z, c.w));
                const float2 r0 = __ffma2_rn(make_float2(a.c1, a.c1), s0, make_float2(-n0.x, -n0.y));
                const float2 r1 = __ffma2_rn(make_float2(a.c1, a.c1), s1, make_float2(-n1.x, -n1.y));
                const bool e0 = x0 > 0, e3 = x0 + 3 < nx - 1;          // x = x0 + 1, x0 + 2 are interior
                *reinterpret_cast<float4*>(a.out + f) =
                    make_float4(e0 ? r0.x : c.x, r0.y, r1.x, e3 ? r1.y : c.w);
#else
                const float cc[4] = {c.x, c.y, c.z, c.w};
                const float am[4] = {zm.x, zm.y, zm.z, zm.w}, ap[4] = {zp.x, zp.y, zp.z, zp.w};
                const float bm[4] = {ym.x, ym.y, ym.z, ym.w}, bp[4] = {yp.x, yp.y, yp.z, yp.w};
                float o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int x = x0 + e;
                    if (x > 0 && x < nx - 1) {
                        float s = am[e] + ap[e];
                        s = s + bm[e];
                        s = s + bp[e];
                        s = s + (e == 0 ? xm : cc[e - 1]);
                        s = s + (e == 3 ? xp : cc[e + 1]);
                        o[e] = fmaf(a.c1, s, -(a.c0 * cc[e]));
                    } else {
                        o[e] = cc[e];
                    }
                }
                *reinterpret_cast<float4*>(a.out + f) = make_float4(o[0], o[1], o[2], o[3]);
#endif
            } else if (act) {
                *reinterpret_cast<float4*>(a.out + f) = c;
            }
            zm = c;
            c = zp;
        }
    }
};

// MRIQ (Parboil ComputeQ): one voxel per thread; k-space staged in 256-entry chunks,
// 2 pi folded into k at staging time, so the inner loop is 3 FMA for the phase, the two MUFU
// ops (__sincosf: FMUL.RZ by 1/2pi, MUFU.SIN, MUFU.COS) and 2 FMA accumulates.  MUFU-bound: 2
// MUFU ops per (voxel, k) take 16 pipe cycles per warp on an SMSP while the loop issues 9
// instructions (ncu: XU 96 %, issue 56 %).
// Measured and not adopted (compile-time KL_MRIQ_P > 0; tools/exp_mriq_mix.py, ncu in
// tools/ncu_mriq_mix.sh): in every group of KL_MRIQ_G k-points the last KL_MRIQ_P take sin/cos
// from FMA-pipe polynomials (sincos_2pi_poly, ~22 issue slots, no MUFU; staged in revolutions).
// Solo, P/G = 1/8 is fastest (1.97 -> 1.82 ms plain grid, 1.98 -> 1.90 ms persistent; at 1/4 the
// XU pipe drops to 71 % but MIO-throttle / not-selected stalls keep the time), but the extra
// issue slots belong to the co-scheduled partner in a Kernelet phase: the model-guided step did
// not get faster (device 10.56-10.93 ms vs 10.41-10.68 ms MUFU-only, same profile), and
// a launch-mode switch (MUFU-only when co-scheduled) would make a co-scheduled MRIQ's result
// depend on its schedule, breaking sliced == unsliced bit-identity.  So P = 0.
#ifndef KL_MRIQ_G
#define KL_MRIQ_G 8
#endif
#ifndef KL_MRIQ_U
#define KL_MRIQ_U 8      // k-point pairs per unrolled group of the FP32x2 loop (4: C5 -0.5 %)
#endif
#ifndef KL_MRIQ_P
#define KL_MRIQ_P 0
#endif
#if KL_MRIQ_P > 0 || defined(KL_MRIQ_SCALAR)
// sin(2 pi t), cos(2 pi t) on the FMA pipe: r = t - rint(t) in [-1/2, 1/2] (rint by the
// 1.5*2^23 rounding trick, exact for |t| < 2^22), then sin = r P(r^2) (degree 5 in r^2) and
// cos = Q(r^2) (degree 6), near-minimax coefficients (Lawson-weighted least squares on
// [-1/2, 1/2], rounded to fp32).  Max abs error in fp32 arithmetic: 7.1e-7 (sin), 4.0e-7 (cos),
// the same order as MUFU.SIN/COS (2^-21 near 0, growing with |t|).
__device__ __forceinline__ void sincos_2pi_poly(float t, float& s, float& c) {
    const float magic = 12582912.0f;                       // 1.5 * 2^23
    const float r = t - ((t + magic) - magic);
    const float u = r * r;
    float ps = fmaf(u, -12.271262168884277f, 41.20539474487305f);
    ps = fmaf(u, ps, -76.5801010131836f);
    ps = fmaf(u, ps, 81.59618377685547f);
    ps = fmaf(u, ps, -41.34142303466797f);
    ps = fmaf(u, ps, 6.283182621002197f);
    s = r * ps;
    float pc = fmaf(u, 6.5296101570129395f, -25.968313217163086f);
    pc = fmaf(u, pc, 60.16783142089844f);
    pc = fmaf(u, pc, -85.45016479492188f);
    pc = fmaf(u, pc, 64.93911743164062f);
    pc = fmaf(u, pc, -19.73920440673828f);
    c = fmaf(u, pc, 1.0f);
}
#endif

struct BodyMRIQ {
    using Params = kl_args_mriq;
    using State = Empty;
#ifdef KL_MRIQ_V2
    static constexpr int kThreads = 256, kChunk = 2, kDynSmem = 0, kMinBlocks = KL_MINB_MRIQ;
#else
    static constexpr int kThreads = 256, kChunk = 1, kDynSmem = 0, kMinBlocks = KL_MINB_MRIQ;
#endif
    static constexpr int kG = KL_MRIQ_G, kP = KL_MRIQ_P;
    static_assert(kP >= 0 && kP < kG, "KL_MRIQ_P in [0, KL_MRIQ_G)");
    __device__ static void init(const Params&, State&, char*) {}
    __device__ static void fini(const Params&, State&, char*) {}
#if KL_MRIQ_P == 0 && !defined(KL_MRIQ_SCALAR)
    // Paired k-points on the sm_100 FP32x2 path (FFMA2 / FMUL2): k-points 2p and 2p+1 of a chunk
    // are staged as sk[2p] = (kx0, kx1, ky0, ky1), sk[2p+1] = (kz0, kz1, phi0, phi1) (x 2 pi), so
    // one FMUL2 + two FFMA2 give both phases and two FFMA2 both accumulates: 13 instructions per
    // two terms instead of 18 (SASS: 2 LDS.128, FMUL2, 4 FFMA2, 2 FMUL.RZ, 4 MUFU).  The MUFU
    // work is unchanged (MRIQ stays MUFU-bound solo); the issue slots it frees are the
    // co-scheduled partner's.  Sums: even and odd k-points accumulate in the two halves (each in
    // k order, one fmaf per term) and meet once at the end -- the order is fixed by num_k alone,
    // so sliced == unsliced stays bit-identical; the fp32 error bound of DESIGN §3 holds (two
    // sums of n_k / 2 terms).
#ifdef KL_MRIQ_V2
    // Two virtual blocks per grid block (a fetched chunk of 2, block_range): every thread runs
    // voxel t of each, so one pair of k-points from shared memory feeds four terms (half the LDS
    // per term); each voxel's arithmetic is exactly the one-voxel path's (sliced == unsliced).
    __device__ static void block_range(const Params& a, State&, char*, uint32_t v0, uint32_t v1) {
        __shared__ float4 sk[256];
        const int i0 = (int)v0 * 256 + threadIdx.x, i1 = i0 + 256;
        const bool l0 = i0 < a.num_x, l1 = v1 > v0 + 1 && i1 < a.num_x;
        const float2 xa = f2(l0 ? __ldg(a.x + i0) : 0.f), ya = f2(l0 ? __ldg(a.y + i0) : 0.f),
                     za = f2(l0 ? __ldg(a.z + i0) : 0.f);
        const float2 xb = f2(l1 ? __ldg(a.x + i1) : 0.f), yb = f2(l1 ? __ldg(a.y + i1) : 0.f),
                     zb = f2(l1 ? __ldg(a.z + i1) : 0.f);
        float2 qra = make_float2(0.f, 0.f), qia = qra, qrb = qra, qib = qra;
        float* skf = reinterpret_cast<float*>(sk);
        for (int k0 = 0; k0 < a.num_k; k0 += 256) {
            const int n = min(256, a.num_k - k0);
            __syncthreads();
            if ((int)threadIdx.x < n) {
                const int k = k0 + threadIdx.x, p = threadIdx.x >> 1, h = threadIdx.x & 1;
                const float sc = 6.28318530717958647692f;
                skf[8 * p + h] = sc * __ldg(a.kx + k);
                skf[8 * p + 2 + h] = sc * __ldg(a.ky + k);
                skf[8 * p + 4 + h] = sc * __ldg(a.kz + k);
                skf[8 * p + 6 + h] = __ldg(a.phimag + k);
            }
            __syncthreads();
            const int np = n >> 1;
            int p = 0;
            for (; p + 4 <= np; p += 4) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float4 aa = sk[2 * (p + j)], bb = sk[2 * (p + j) + 1];
                    pair(aa, bb, xa, ya, za, qra, qia);
                    pair(aa, bb, xb, yb, zb, qrb, qib);
                }
            }
            for (; p < np; ++p) {
                const float4 aa = sk[2 * p], bb = sk[2 * p + 1];
                pair(aa, bb, xa, ya, za, qra, qia);
                pair(aa, bb, xb, yb, zb, qrb, qib);
            }
            if (n & 1) {
                const float4 aa = sk[2 * np], bb = sk[2 * np + 1];
                tail(aa, bb, xa.x, ya.x, za.x, qra, qia);
                tail(aa, bb, xb.x, yb.x, zb.x, qrb, qib);
            }
        }
        if (l0) {
            a.qr[i0] = qra.x + qra.y;
            a.qi[i0] = qia.x + qia.y;
        }
        if (l1) {
            a.qr[i1] = qrb.x + qrb.y;
            a.qi[i1] = qib.x + qib.y;
        }
    }
    __device__ static __forceinline__ float2 f2(float v) { return make_float2(v, v); }
    __device__ static __forceinline__ void tail(const float4 aa, const float4 bb, float x, float y, float z,
                                                float2& qr, float2& qi) {
        const float t = fmaf(aa.x, x, fmaf(aa.z, y, bb.x * z));
        float sn, cs;
        __sincosf(t, &sn, &cs);
        qr.x = fmaf(bb.z, cs, qr.x);
        qi.x = fmaf(bb.z, sn, qi.x);
    }
#else
    __device__ static void block(const Params& a, State&, char*, uint32_t vb) {
        __shared__ float4 sk[256];
        const int i = (int)vb * 256 + threadIdx.x;
        const bool live = i < a.num_x;
        const float x = live ? __ldg(a.x + i) : 0.f, y = live ? __ldg(a.y + i) : 0.f,
                    z = live ? __ldg(a.z + i) : 0.f;
        const float2 x2 = make_float2(x, x), y2 = make_float2(y, y), z2 = make_float2(z, z);
        float2 qr = make_float2(0.f, 0.f), qi = make_float2(0.f, 0.f);
        float* skf = reinterpret_cast<float*>(sk);
        for (int k0 = 0; k0 < a.num_k; k0 += 256) {
            const int n = min(256, a.num_k - k0);
            __syncthreads();
            if ((int)threadIdx.x < n) {
                const int k = k0 + threadIdx.x, p = threadIdx.x >> 1, h = threadIdx.x & 1;
                const float sc = 6.28318530717958647692f;
                skf[8 * p + h] = sc * __ldg(a.kx + k);
                skf[8 * p + 2 + h] = sc * __ldg(a.ky + k);
                skf[8 * p + 4 + h] = sc * __ldg(a.kz + k);
                skf[8 * p + 6 + h] = __ldg(a.phimag + k);
            }
            __syncthreads();
            const int np = n >> 1;
            int p = 0;
            for (; p + KL_MRIQ_U <= np; p += KL_MRIQ_U) {
#pragma unroll
                for (int j = 0; j < KL_MRIQ_U; ++j) pair(sk[2 * (p + j)], sk[2 * (p + j) + 1], x2, y2, z2, qr, qi);
            }
            for (; p < np; ++p) pair(sk[2 * p], sk[2 * p + 1], x2, y2, z2, qr, qi);
            if (n & 1) {                                    // odd tail: the even half's term
                const float4 aa = sk[2 * np], bb = sk[2 * np + 1];
                const float t = fmaf(aa.x, x, fmaf(aa.z, y, bb.x * z));
                float sn, cs;
                __sincosf(t, &sn, &cs);
                qr.x = fmaf(bb.z, cs, qr.x);
                qi.x = fmaf(bb.z, sn, qi.x);
            }
        }
        if (live) {
            a.qr[i] = qr.x + qr.y;
            a.qi[i] = qi.x + qi.y;
        }
    }
#endif
    __device__ static __forceinline__ void pair(const float4 aa, const float4 bb, const float2 x2, const float2 y2,
                                                const float2 z2, float2& qr, float2& qi) {
        float2 t = __fmul2_rn(make_float2(bb.x, bb.y), z2);
        t = __ffma2_rn(make_float2(aa.z, aa.w), y2, t);
        t = __ffma2_rn(make_float2(aa.x, aa.y), x2, t);
        float s0, c0, s1, c1;
        __sincosf(t.x, &s0, &c0);
        __sincosf(t.y, &s1, &c1);
        const float2 ph = make_float2(bb.z, bb.w);
        qr = __ffma2_rn(ph, make_float2(c0, c1), qr);
        qi = __ffma2_rn(ph, make_float2(s0, s1), qi);
    }
#else
    __device__ static __forceinline__ void term(const float4 q, float x, float y, float z, bool poly,
                                                float& qr, float& qi) {
        const float t = fmaf(q.x, x, fmaf(q.y, y, q.z * z));
        float sn, cs;
        if (poly) sincos_2pi_poly(t, sn, cs);
        else __sincosf(t, &sn, &cs);
        qr = fmaf(q.w, cs, qr);
        qi = fmaf(q.w, sn, qi);
    }
    __device__ static void block(const Params& a, State&, char*, uint32_t vb) {
        __shared__ float4 sk[256];   // (kx, ky, kz) x 2 pi (MUFU terms) or x 1 (polynomial terms), phiMag
        const int i = (int)vb * 256 + threadIdx.x;
        const bool live = i < a.num_x;
        const float x = live ? __ldg(a.x + i) : 0.f, y = live ? __ldg(a.y + i) : 0.f,
                    z = live ? __ldg(a.z + i) : 0.f;
        float qr = 0.f, qi = 0.f;
        for (int k0 = 0; k0 < a.num_k; k0 += 256) {
            const int n = min(256, a.num_k - k0);
            const int n_full = n - n % kG;                  // whole groups; the tail is all MUFU
            __syncthreads();
            if ((int)threadIdx.x < n) {
                const int k = k0 + threadIdx.x;
                const bool poly = (int)threadIdx.x < n_full && (int)threadIdx.x % kG >= kG - kP;
                const float sc = poly ? 1.0f : 6.28318530717958647692f;
                sk[threadIdx.x] = make_float4(sc * __ldg(a.kx + k), sc * __ldg(a.ky + k),
                                              sc * __ldg(a.kz + k), __ldg(a.phimag + k));
            }
            __syncthreads();
            int k = 0;
            for (; k < n_full; k += kG) {
#pragma unroll
                for (int j = 0; j < kG; ++j) term(sk[k + j], x, y, z, j >= kG - kP, qr, qi);
            }
            for (; k < n; ++k) term(sk[k], x, y, z, false, qr, qi);
        }
        if (live) {
            a.qr[i] = qr;
            a.qi[i] = qi;
        }
    }
#endif
};

// BS (SDK BlackScholes): 128 threads x 5 float4 = 2560 options per block.
// The SDK sample's formula with the hardware approximations (MUFU ex2/lg2/rcp, ~2 ulp): BS is
// issue-bound at paper size, and the result stays far inside the normwise 1e-5 tolerance.
#ifdef KL_BS_SCALAR
__device__ __forceinline__ float cnd_f(float d) {
    const float A1 = 0.31938153f, A2 = -0.356563782f, A3 = 1.781477937f, A4 = -1.821255978f,
                A5 = 1.330274429f, RSQRT2PI = 0.39894228040143267793994605993438f;
    float K = __frcp_rn(1.0f + 0.2316419f * fabsf(d));
    float c = RSQRT2PI * __expf(-0.5f * d * d) * (K * (A1 + K * (A2 + K * (A3 + K * (A4 + K * A5)))));
    return d > 0.f ? 1.0f - c : c;
}
__device__ __forceinline__ void bs_one(float S, float X, float T, float R, float V, float& call, float& put) {
    float sqrtT = sqrtf(T);
    float d1 = __fdividef(__logf(__fdividef(S, X)) + (R + 0.5f * V * V) * T, V * sqrtT);
    float d2 = d1 - V * sqrtT;
    float c1 = cnd_f(d1), c2 = cnd_f(d2);
    float e = __expf(-R * T);
    call = S * c1 - X * e * c2;
    put = X * e * (1.0f - c2) - S * (1.0f - c1);
}
#endif
#ifndef KL_BS_SCALAR
// Two options at a time on the sm_100 FP32x2 path (FFMA2 / FMUL2 / FADD2): the arithmetic of
// bs_one in pairs, the MUFU-based functions (sqrtf, __fdividef, __logf, __expf, __frcp_rn) per
// option.  BS was issue-bound (ncu: issue 82 %, fma pipe 49 %); the pairs halve its FP32 issue
// slots.  Same operations per option as bs_one up to contraction choices (normwise tolerance).
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 cnd_f2(float2 d) {
    const float A1 = 0.31938153f, A2 = -0.356563782f, A3 = 1.781477937f, A4 = -1.821255978f,
                A5 = 1.330274429f, RSQRT2PI = 0.39894228040143267793994605993438f;
    const float2 den = __ffma2_rn(f2(0.2316419f), make_float2(fabsf(d.x), fabsf(d.y)), f2(1.0f));
    const float2 K = make_float2(__frcp_rn(den.x), __frcp_rn(den.y));
    const float2 dd = __fmul2_rn(__fmul2_rn(f2(-0.5f), d), d);
    const float2 ex = make_float2(__expf(dd.x), __expf(dd.y));
    float2 p = __ffma2_rn(K, f2(A5), f2(A4));
    p = __ffma2_rn(K, p, f2(A3));
    p = __ffma2_rn(K, p, f2(A2));
    p = __ffma2_rn(K, p, f2(A1));
    const float2 c = __fmul2_rn(__fmul2_rn(f2(RSQRT2PI), ex), __fmul2_rn(K, p));
    return make_float2(d.x > 0.f ? 1.0f - c.x : c.x, d.y > 0.f ? 1.0f - c.y : c.y);
}
__device__ __forceinline__ void bs_two(float2 S, float2 X, float2 T, float R, float V, float2& call, float2& put) {
    const float2 sqrtT = make_float2(sqrtf(T.x), sqrtf(T.y));
    const float2 lg = make_float2(__logf(__fdividef(S.x, X.x)), __logf(__fdividef(S.y, X.y)));
    const float2 vs = __fmul2_rn(f2(V), sqrtT);
    const float2 num = __ffma2_rn(f2(R + 0.5f * V * V), T, lg);
    const float2 d1 = make_float2(__fdividef(num.x, vs.x), __fdividef(num.y, vs.y));
    const float2 d2 = __fadd2_rn(d1, make_float2(-vs.x, -vs.y));
    const float2 c1 = cnd_f2(d1), c2 = cnd_f2(d2);
    const float2 rt = __fmul2_rn(f2(-R), T);
    const float2 xe = __fmul2_rn(X, make_float2(__expf(rt.x), __expf(rt.y)));
    const float2 u = __fmul2_rn(xe, c2);
    call = __ffma2_rn(S, c1, make_float2(-u.x, -u.y));
    const float2 v = __fmul2_rn(xe, __fadd2_rn(f2(1.0f), make_float2(-c2.x, -c2.y)));
    put = __ffma2_rn(make_float2(-S.x, -S.y), __fadd2_rn(f2(1.0f), make_float2(-c1.x, -c1.y)), v);
}
#endif
struct BodyBS {
    using Params = kl_args_bs;
    using State = Empty;
    static constexpr int kThreads = 128, kChunk = 1, kDynSmem = 0, kMinBlocks = KL_MINB_BS;
    __device__ static void init(const Params&, State&, char*) {}
    __device__ static void fini(const Params&, State&, char*) {}
    __device__ static void block(const Params& a, State&, char*, uint32_t vb) {
        const int64_t n4 = a.n / 4;
        const float4* S = reinterpret_cast<const float4*>(a.S);
        const float4* X = reinterpret_cast<const float4*>(a.X);
        const float4* T = reinterpret_cast<const float4*>(a.T);
        float4* C = reinterpret_cast<float4*>(a.call);
        float4* P = reinterpret_cast<float4*>(a.put);
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            int64_t i = (int64_t)vb * 640 + j * 128 + threadIdx.x;
            if (i >= n4) break;
            float4 s = __ldg(S + i), x = __ldg(X + i), t = __ldg(T + i), c, p;
#ifdef KL_BS_SCALAR
            bs_one(s.x, x.x, t.x, a.R, a.V, c.x, p.x);
            bs_one(s.y, x.y, t.y, a.R, a.V, c.y, p.y);
            bs_one(s.z, x.z, t.z, a.R, a.V, c.z, p.z);
            bs_one(s.w, x.w, t.w, a.R, a.V, c.w, p.w);
#else
            float2 c0, p0, c1, p1;
            bs_two(make_float2(s.x, s.y), make_float2(x.x, x.y), make_float2(t.x, t.y), a.R, a.V, c0, p0);
            bs_two(make_float2(s.z, s.w), make_float2(x.z, x.w), make_float2(t.z, t.w), a.R, a.V, c1, p1);
            c = make_float4(c0.x, c0.y, c1.x, c1.y);
            p = make_float4(p0.x, p0.y, p1.x, p1.y);
#endif
            C[i] = c;
            P[i] = p;
        }
    }
};

// TEA: 32 cycles per 64-bit block; uint4 = two blocks; 1280 blocks per thread block.
__device__ __forceinline__ void tea_enc(uint32_t& v0, uint32_t& v1, uint32_t k0, uint32_t k1, uint32_t k2, uint32_t k3) {
    uint32_t sum = 0;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
        sum += 0x9E3779B9u;
        v0 += ((v1 << 4) + k0) ^ (v1 + sum) ^ ((v1 >> 5) + k1);
        v1 += ((v0 << 4) + k2) ^ (v0 + sum) ^ ((v0 >> 5) + k3);
    }
}
struct BodyTEA {
    using Params = kl_args_tea;
    using State = Empty;
    static constexpr int kThreads = 128, kChunk = 1, kDynSmem = 0, kMinBlocks = 16;
    __device__ static void init(const Params&, State&, char*) {}
    __device__ static void fini(const Params&, State&, char*) {}
    __device__ static void block(const Params& a, State&, char*, uint32_t vb) {
        const int64_t n2 = a.n / 2;
        const uint4* in = reinterpret_cast<const uint4*>(a.in);
        uint4* out = reinterpret_cast<uint4*>(a.out);
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            int64_t i = (int64_t)vb * 640 + j * 128 + threadIdx.x;
            if (i >= n2) break;
            uint4 v = __ldg(in + i);
            tea_enc(v.x, v.y, a.key[0], a.key[1], a.key[2], a.key[3]);
            tea_enc(v.z, v.w, a.key[0], a.key[1], a.key[2], a.key[3]);
            out[i] = v;
        }
    }
};

// MatrixAdd: 16x16 threads per block over a (n/16) x (n/16) grid.
struct BodyMATADD {
    using Params = kl_args_matadd;
    using State = Empty;
    static constexpr int kThreads = 256, kChunk = 1, kDynSmem = 0, kMinBlocks = 8;
    __device__ static void init(const Params&, State&, char*) {}
    __device__ static void fini(const Params&, State&, char*) {}
    __device__ static void block(const Params& a, State&, char*, uint32_t vb) {
        const int g = a.n / 16, bx = vb % g, by = vb / g;
        if (by >= g) return;                      // a grid larger than the matrix
        const int i = (by * 16 + (threadIdx.x >> 4)) * a.n + bx * 16 + (threadIdx.x & 15);
        a.C[i] = a.A[i] + a.B[i];
    }
};

// Synthetic streaming kernel: 4 float4 per thread, `fmas` dependent FMAs each.
struct BodySYNTH {
    using Params = kl_args_synth;
    using State = Empty;
    static constexpr int kThreads = 256, kChunk = 1, kDynSmem = 0, kMinBlocks = 8;
    __device__ static void init(const Params&, State&, char*) {}
    __device__ static void fini(const Params&, State&, char*) {}
    __device__ static void block(const Params& a, State&, char*, uint32_t vb) {
        const int64_t n4 = a.n / 4;
        const float4* x = reinterpret_cast<const float4*>(a.x);
        float4* y = reinterpret_cast<float4*>(a.y);
        float4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int64_t i = (int64_t)vb * 1024 + j * 256 + threadIdx.x;
            v[j] = i < n4 ? __ldg(x + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        for (int c = 0; c < a.fmas; ++c) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                v[j].x = fmaf(v[j].x, a.a, a.b); v[j].y = fmaf(v[j].y, a.a, a.b);
                v[j].z = fmaf(v[j].z, a.a, a.b); v[j].w = fmaf(v[j].w, a.a, a.b);
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int64_t i = (int64_t)vb * 1024 + j * 256 + threadIdx.x;
            if (i < n4) y[i] = v[j];
        }
    }
};

}  // namespace

// MM lives in kl_mm.cu (tcgen05); these are its entry points.
int kl_mm_info(KlKindInfo* o);
int kl_mm_prepare(const void* args, uint32_t bytes, uint32_t grid, void* blob, uint32_t cap);
int kl_mm_launch_persistent(const void* blob, const KlLaunch& L, uint32_t grid, void* stream);
int kl_mm_launch_plain(const void* blob, uint32_t offset, uint32_t n, void* stream);

#define KL_DISPATCH(kind, FN, ...)                                   \
    switch (kind) {                                                  \
        case KL_PC: return FN<BodyPC>(__VA_ARGS__);                  \
        case KL_SAD: return FN<BodySAD>(__VA_ARGS__);                \
        case KL_SPMV: return FN<BodySPMV>(__VA_ARGS__);              \
        case KL_ST: return FN<BodyST>(__VA_ARGS__);                  \
        case KL_MRIQ: return FN<BodyMRIQ>(__VA_ARGS__);              \
        case KL_BS: return FN<BodyBS>(__VA_ARGS__);                  \
        case KL_TEA: return FN<BodyTEA>(__VA_ARGS__);                \
        case KL_MATADD: return FN<BodyMATADD>(__VA_ARGS__);          \
        case KL_SYNTH: return FN<BodySYNTH>(__VA_ARGS__);            \
        default: return -1;                                          \
    }

static const uint32_t kArgBytes[KL_NKINDS] = {
    sizeof(kl_args_pc), sizeof(kl_args_sad), sizeof(kl_args_spmv), sizeof(kl_args_st),
    sizeof(kl_args_mm), sizeof(kl_args_mriq), sizeof(kl_args_bs), sizeof(kl_args_tea),
    sizeof(kl_args_matadd), sizeof(kl_args_synth)};

uint32_t kl_args_size(int kind) { return (kind >= 0 && kind < KL_NKINDS) ? kArgBytes[kind] : 0u; }

template <class Body>
int preload_of() {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k_plain<Body>);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaFuncGetAttributes(&fa, k_persistent<Body>);
}

int kl_dev_kind_info(int kind, KlKindInfo* out) {
    if (kind == KL_MM) return kl_mm_info(out);
    KL_DISPATCH(kind, info_of, out);
}

int kl_dev_prepare(int kind, const void* args, uint32_t bytes, uint32_t grid, void* blob, uint32_t cap) {
    if (kind < 0 || kind >= KL_NKINDS || bytes != kArgBytes[kind]) return -1;
    if (kind == KL_MM) return kl_mm_prepare(args, bytes, grid, blob, cap);
    if (bytes > cap) return -1;
    if (kind == KL_ST && (reinterpret_cast<const kl_args_st*>(args)->nx % 4)) return -1;   // float4 rows
    std::memcpy(blob, args, bytes);
    return 0;
}

int kl_dev_launch_persistent(int kind, const void* blob, const KlLaunch& L, uint32_t grid, void* stream) {
    if (kind == KL_MM) return kl_mm_launch_persistent(blob, L, grid, stream);
    KL_DISPATCH(kind, launch_persistent, blob, L, grid, stream);
}

int kl_dev_launch_plain(int kind, const void* blob, uint32_t offset, uint32_t n, void* stream) {
    if (kind == KL_MM) return kl_mm_launch_plain(blob, offset, n, stream);
    KL_DISPATCH(kind, launch_plain, blob, offset, n, stream);
}

// Arrival clock (online arrivals): one thread sleeps until `ns` after its own start
// (device %globaltimer), then stamps the release time; the caller records its kernel's ready
// event after it on the same stream.
__global__ void k_delay(unsigned long long ns, unsigned long long* stamp) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 >= ns) break;
        __nanosleep(1000);
    }
    if (stamp) *stamp = t;
}

// Resident arrival clock: one thread releases n arrivals at cumulative device-time gaps.
__global__ void k_arrival_clock(const unsigned long long* gaps, unsigned long long* stamps, volatile uint32_t* flags,
                                uint32_t n) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    unsigned long long due = t;
    for (uint32_t i = 0; i < n; ++i) {
        due += gaps[i];
        for (;;) {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t >= due) break;
            __nanosleep(500);
        }
        stamps[i] = t;
        __threadfence_system();
        flags[i] = 1u;
        __threadfence_system();
    }
}

int kl_dev_arrival_clock(const unsigned long long* gaps, unsigned long long* stamps, uint32_t* flags, uint32_t n,
                         void* stream) {
    k_arrival_clock<<<1, 1, 0, (cudaStream_t)stream>>>(gaps, stamps, flags, n);
    return (int)cudaGetLastError();
}

__global__ void k_wait_flag(const volatile uint32_t* flag, unsigned long long* stamp) {
    if (flag)
        while (*flag == 0u) __nanosleep(500);
    if (stamp) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        *stamp = t;
    }
}

int kl_dev_wait_flag(const volatile uint32_t* flag, unsigned long long* stamp, void* stream) {
    k_wait_flag<<<1, 1, 0, (cudaStream_t)stream>>>(flag, stamp);
    return (int)cudaGetLastError();
}

int kl_dev_delay(unsigned long long ns, unsigned long long* stamp, void* stream) {
    k_delay<<<1, 1, 0, (cudaStream_t)stream>>>(ns, stamp);
    return (int)cudaGetLastError();
}

// Initialise slice control blocks from a (host-mapped) list of (slot, len, gen) triples; optionally
// reset the completion counters (kl_counters layout; t_start = INT64_MAX).
__global__ void k_ctl_init(KlCtl* pool, const uint32_t* slots_lens, int n, unsigned long long* counters) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (counters && t < 5) counters[t] = (t == 2) ? 0x7fffffffffffffffull : 0ull;
    for (int i = t; i < n; i += gridDim.x * blockDim.x) {
        KlCtl* c = pool + slots_lens[3 * i];
        c->word = kl_w_make(0u, 0u, 0u, false);
        c->len = slots_lens[3 * i + 1];
        // count-preserving: a late block of the slot's previous kernel may have a stray join
        // pending its undo
        unsigned long long cur = atomicAdd(&c->join, 0ull);
        for (;;) {
            const unsigned long long nw = (cur & 0xffffffffull) | kl_j_make(kl_ticket(slots_lens[3 * i + 2], 0u), false);
            const unsigned long long prev = atomicCAS(&c->join, cur, nw);
            if (prev == cur) break;
            cur = prev;
        }
        c->tune = 0ull;
        c->drained = 0;
        c->admitted = 0;
        c->executed = 0;
        c->base = 0;
        c->t0 = ~0ull;
        c->stop_req = 0ull;
    }
}

int kl_dev_ctl_init(KlCtl* pool, const uint32_t* slots_lens, int n, unsigned long long* counters, void* stream) {
    if (n <= 0 && !counters) return 0;
    const int blocks = n > 0 ? (n + 255) / 256 : 1;
    k_ctl_init<<<blocks, 256, 0, (cudaStream_t)stream>>>(pool, slots_lens, n, counters);
    return (int)cudaGetLastError();
}

// Load every kernel of this file now (called by kl_create): with lazy module loading, a first
// launch during scheduling would synchronise the device behind unrelated streams.
int kl_dev_preload() {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k_ctl_init);
    if (e != cudaSuccess) return (int)e;
    e = cudaFuncGetAttributes(&fa, k_delay);
    if (e != cudaSuccess) return (int)e;
    e = cudaFuncGetAttributes(&fa, k_arrival_clock);
    if (e != cudaSuccess) return (int)e;
    e = cudaFuncGetAttributes(&fa, k_wait_flag);
    if (e != cudaSuccess) return (int)e;
    for (int kind = 0; kind < KL_NKINDS; ++kind) {
        if (kind == KL_MM) continue;
        int rc = [&]() -> int { KL_DISPATCH(kind, preload_of); }();
        if (rc) return rc;
    }
    return 0;
}

