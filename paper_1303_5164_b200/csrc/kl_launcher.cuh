// kl_launcher.cuh -- the persistent slice launcher shared by every kernel body (product path).
//
// Slicing: a slice is a contiguous range of a kernel's thread blocks launched with
// its block index rectified by an offset.  On B200 a phase launches ONE persistent grid per
// kernel (cap x n_SM blocks); each admitted block pulls virtual block ids from the kernel's
// slice control word (KlCtl) and runs Body::block(vb).  Occupancy control is a per-SM admission
// cap read from %smid.  When a kernel drains, its first block to notice stops the partner's
// launch at the partner's next slice boundary (Alg.1 l.9).  Included by kl_kernels.cu and
// kl_mm.cu (header-only so no relocatable device code is needed).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "kl_internal.h"

namespace {

__device__ __forceinline__ uint32_t smid_u32() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ------------------------------------------------------------------------------------------
// Slice launcher.
// ------------------------------------------------------------------------------------------
// Stop the partner's current launch at its first slice boundary at or after its current
// position (Alg.1 l.9: the co-schedule is kept only while both kernels still have blocks).
__device__ void stop_at_boundary(KlCtl* p, uint32_t pstart, uint32_t pslice) {
    unsigned long long old = atomicAdd(&p->word, 0ull);
    for (;;) {
        if (old >> 63) return;
        uint32_t nx = (uint32_t)old;
        uint32_t rel = nx > pstart ? nx - pstart : 0u;
        uint32_t sl = pslice ? pslice : 1u;
        // first slice boundary at or after the current position, but at least one slice into
        // the launch: a co-schedule runs a slice of each kernel, even when the
        // partner's blocks had not been dispatched yet when this kernel drained
        unsigned long long nsl = (unsigned long long)(rel + sl - 1) / sl;
        if (nsl == 0) nsl = 1;
        unsigned long long sa = (unsigned long long)pstart + nsl * sl;
        if (sa < nx) sa = nx;
        if (sa > 0x7fffffffull) sa = 0x7fffffffull;
        unsigned long long nw = (old & 0xffffffffull) | (sa << 32) | (1ull << 63);
        unsigned long long prev = atomicCAS(&p->word, old, nw);
        if (prev == old) return;
        old = prev;
    }
}

__device__ void finalize_launch(const KlLaunch& L, uint32_t len) {
    KlCtl* ctl = L.ctl;
    __threadfence();
    unsigned long long w = atomicAdd(&ctl->word, 0ull);
    uint32_t lim = len;
    if (w >> 63) lim = min(lim, (uint32_t)((w >> 32) & 0x7fffffffu));
    uint32_t executed = atomicExch(&ctl->executed, 0u);
    uint32_t admitted = atomicExch(&ctl->admitted, 0u);
    uint32_t mx = 0;
    for (uint32_t s = 0; s < L.n_sms && s < KL_MAX_SMS; ++s) {
        mx = max(mx, ctl->sm_hwm[s]);
        ctl->sm_hwm[s] = 0;
    }
    unsigned long long t0 = atomicExch(&ctl->t0, ~0ull);
    unsigned long long t1 = gtimer();
    atomicExch(&ctl->word, (unsigned long long)lim);   // next = lim, stop cleared
    atomicExch(&ctl->exited, 0u);
    const bool exh = (lim == len);
    if (L.counters) {
        atomicAdd(&L.counters[1], (unsigned long long)executed);
        if (exh) {
            atomicAdd(&L.counters[0], 1ull);
            atomicAdd(&L.counters[4], L.tag);
        }
        if (admitted) atomicMin(reinterpret_cast<long long*>(&L.counters[2]), (long long)t0);
        atomicMax(reinterpret_cast<long long*>(&L.counters[3]), (long long)t1);
    }
    KlLaunchRec* r = L.rec;
    if (r) {
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

template <class Body>
__global__ void __launch_bounds__(Body::kThreads)
k_persistent(const __grid_constant__ typename Body::Params P, const __grid_constant__ KlLaunch L) {
    extern __shared__ __align__(1024) char dsmem[];
    __shared__ uint32_t s_vb[2], s_end[2], s_adm;
    KlCtl* ctl = L.ctl;
    const uint32_t len = ctl->len;
    uint32_t sm = 0;
    if (threadIdx.x == 0) {
        uint32_t adm = 1;
        sm = smid_u32();
        if (L.cap) {
            uint32_t c = atomicAdd(&ctl->sm_count[sm], 1u);
            if (c >= L.cap) {
                atomicSub(&ctl->sm_count[sm], 1u);
                adm = 0;
            } else {
                atomicMax(&ctl->sm_hwm[sm], c + 1);
            }
        }
        if (adm) {
            atomicAdd(&ctl->admitted, 1u);
            atomicMin(&ctl->t0, gtimer());
        }
        s_adm = adm;
    }
    __syncthreads();
    if (s_adm) {
        typename Body::State st;
        Body::init(P, st, dsmem);
        uint32_t nexec = 0;
        for (uint32_t it = 0;; ++it) {
            if (threadIdx.x == 0) {
                unsigned long long old = atomicAdd(&ctl->word, (unsigned long long)L.chunk);
                uint32_t vb = (uint32_t)old;
                uint32_t lim = len;
                if (old >> 63) lim = min(lim, (uint32_t)((old >> 32) & 0x7fffffffu));
                uint32_t end = vb < lim ? min(vb + L.chunk, lim) : vb;
                if (vb >= len && lim == len && L.partner) {
                    if (atomicCAS(&ctl->drained, 0u, 1u) == 0u)
                        stop_at_boundary(L.partner, L.partner_start, L.partner_slice);
                }
                s_vb[it & 1] = vb;
                s_end[it & 1] = end;
            }
            __syncthreads();
            const uint32_t vb = s_vb[it & 1], end = s_end[it & 1];
            if (vb >= end) break;
            for (uint32_t v = vb; v < end; ++v) {
                Body::block(P, st, dsmem, v);
                if (L.audit && threadIdx.x == 0) atomicAdd(L.audit + v, 1u);
            }
            nexec += end - vb;
        }
        Body::fini(P, st, dsmem);
        if (threadIdx.x == 0) {
            atomicAdd(&ctl->executed, nexec);
            if (L.cap) atomicSub(&ctl->sm_count[sm], 1u);
        }
    }
    if (threadIdx.x == 0) {
        __threadfence();
        uint32_t e = atomicAdd(&ctl->exited, 1u);
        if (e == gridDim.x - 1) finalize_launch(L, len);
    }
}

// Plain grid: blockIdx rectified by the slice offset.
template <class Body>
__global__ void __launch_bounds__(Body::kThreads)
k_plain(const __grid_constant__ typename Body::Params P, uint32_t offset) {
    extern __shared__ __align__(1024) char dsmem[];
    typename Body::State st;
    Body::init(P, st, dsmem);
    Body::block(P, st, dsmem, offset + blockIdx.x);
    Body::fini(P, st, dsmem);
}

template <class Body>
int info_of(KlKindInfo* o) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k_persistent<Body>);
    if (e != cudaSuccess) return (int)e;
    if (Body::kDynSmem > 48 * 1024) {
        e = cudaFuncSetAttribute(k_persistent<Body>, cudaFuncAttributeMaxDynamicSharedMemorySize, Body::kDynSmem);
        if (e != cudaSuccess) return (int)e;
        e = cudaFuncSetAttribute(k_plain<Body>, cudaFuncAttributeMaxDynamicSharedMemorySize, Body::kDynSmem);
        if (e != cudaSuccess) return (int)e;
    }
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

template <class Body>
int launch_plain(const void* blob, uint32_t offset, uint32_t n, void* stream) {
    const auto& P = *reinterpret_cast<const typename Body::Params*>(blob);
    if (n == 0) return 0;
    k_plain<Body><<<n, Body::kThreads, Body::kDynSmem, (cudaStream_t)stream>>>(P, offset);
    return (int)cudaGetLastError();
}


}  // namespace
