// common.cuh -- device helpers shared by the translation units of libtlb.so
// (tlb.cu: single-step kernels and the C ABI; tb2.cu: the two-step kernel).
#pragma once
#include <cuda_runtime.h>

#include "../../include/tlb.h"
#include "d2q37.cuh"

// ------------------------------------------------- peer mailbox protocol --
// (tlb_peer.cuh: the single-step ring; tb2.cu: the two-step ring)
// Default bound of the border blocks' wait; tlb_peer_set_timeout sets it per
// peer object (the host passes its fabric timeout).
#define TLB_PEER_TIMEOUT_NS 5000000000ull

// mailbox layout (u64): [0..7] value published by the neighbour in direction
// d, [8] border-block counter, [9] sticky failure flag, [10] work counter.  A published value
// carries the neighbour's step count (bits 0..39), the step tag = its step
// number + 1 (bits 40..62; runtime.py:151-154's step check) and, in bit 63,
// "I failed" (a timed-out rank poisons what it publishes, so its neighbours
// stop too instead of using halos that were never written).
#define TLB_MB_COUNTER 8
#define TLB_MB_STICKY 9
#define TLB_MB_WORK 10     /* the ring two-step kernel's work-item counter */
#define TLB_MB_CTR_MASK ((1ull << 40) - 1)
#define TLB_MB_TAG_SHIFT 40
#define TLB_MB_TAG_MASK ((1ull << 23) - 1)
#define TLB_MB_POISON (1ull << 63)

namespace tlb {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// --------------------------------------------------------- device helpers --
struct Fld {
    double *base;
    long long sl, sx, sy;
    int Lx, Ly, Hx, Hy;
};

static Fld mkfld(const TlbField *f) {
    Fld d;
    d.base = f->base;
    d.sl = f->sl; d.sx = f->sx; d.sy = f->sy;
    d.Lx = f->Lx; d.Ly = f->Ly; d.Hx = f->Hx; d.Hy = f->Hy;
    return d;
}

static Phys mkphys(const TlbParams *p) {
    // exactly the reference's host-side expressions (kernels.py:130-133, 145)
    Phys P;
    P.K1 = p->tau * p->gx;
    P.K2 = p->tau * p->gy;
    double g2 = p->gx * p->gx + p->gy * p->gy;
    P.K3 = p->tau * p->tau * g2 / 2.0;
    P.omega = p->dt / p->tau;
    P.Tbot = p->Twall_bot;
    P.Ttop = p->Twall_top;
    P.order = p->order;
    return P;
}

__device__ __forceinline__ void report(TlbStatus *st, unsigned bits, int x, int y, int step) {
    if (!bits || !st) return;
    unsigned old = atomicOr(&st->flags, bits);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if ((bits >> k & 1u) && !(old >> k & 1u)) {
            st->site_x[k] = x;
            st->site_y[k] = y;
            st->step = step;
        }
    }
}

// Block-level count of negative populations: one atomic per CTA that saw
// any (count_negative, monitoring only).
__device__ __forceinline__ void count_neg_n(TlbStatus *st, unsigned n) {
    n = __reduce_add_sync(0xffffffffu, n);
    if (__syncthreads_or(n != 0)) {
        __shared__ unsigned warp_n[32];
        if ((threadIdx.x & 31) == 0) warp_n[threadIdx.x >> 5] = n;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned t = 0;
            for (unsigned w = 0; w < (blockDim.x + 31) / 32; ++w) t += warp_n[w];
            if (t) atomicAdd(&st->negatives, (unsigned long long)t);
        }
    }
}

// Negatives test in one integer op per value: OR the high words; only a
// result with the sign bit set (v < 0, -0.0 or a negative NaN) needs the
// exact count (v < 0.0, kernels.py:227-229).
__device__ __forceinline__ unsigned sign_or(unsigned acc, double v) {
    return acc | (unsigned)__double2hiint(v);
}

__device__ __forceinline__ void count_neg(TlbStatus *st, const double (&f)[Q], bool active) {
    unsigned n = 0;
    if (active) {
#pragma unroll
        for (int l = 0; l < Q; ++l) n += f[l] < 0.0;
    }
    count_neg_n(st, n);
}

// Source coordinate of population l's pull for site (x, y) with implicit
// halos (TLB_F_WRAP_X / WRAP_Y / CLAMP_Y), else the halo memory itself.
__device__ __forceinline__ int src_x(int x, int cx, const Fld &s, int flags) {
    int xs = x - cx;
    if (flags & TLB_F_WRAP_X) {
        if (xs < s.Hx) xs += s.Lx;
        else if (xs >= s.Hx + s.Lx) xs -= s.Lx;
    }
    return xs;
}
__device__ __forceinline__ int src_y(int y, int cy, const Fld &s, int flags) {
    int ys = y - cy;
    if (flags & TLB_F_WRAP_Y) {
        if (ys < s.Hy) ys += s.Ly;
        else if (ys >= s.Hy + s.Ly) ys -= s.Ly;
    } else {
        if ((flags & TLB_F_CLAMP_BOT) && ys < s.Hy) ys = s.Hy;
        if ((flags & TLB_F_CLAMP_TOP) && ys >= s.Hy + s.Ly) ys = s.Hy + s.Ly - 1;
    }
    return ys;
}

// COH: coherent L2 loads (ld.global.cg) for data other GPUs write while the
// kernel runs (the peer step's halos); else the read-only path (__ldg).
template <int l, bool COH = false>
__device__ __forceinline__ void load_one(double (&f)[Q], const Fld &s, int x, int y,
                                         bool gather, bool implicit, int flags) {
    int xs = x, ys = y;
    if (gather) {
        if (implicit) {
            xs = src_x(x, CX(l), s, flags);
            ys = src_y(y, CY(l), s, flags);
        } else {
            xs = x - CX(l);
            ys = y - CY(l);
        }
    }
    const double *p = s.base + (long long)l * s.sl + (long long)xs * s.sx + (long long)ys * s.sy;
    f[l] = COH ? __ldcg(p) : __ldg(p);
}

template <bool COH, int... Ls>
struct LoadSeq {
    __device__ __forceinline__ static void run(double (&f)[Q], const Fld &s, int x, int y,
                                               bool gather, bool implicit, int flags) {
        (load_one<Ls, COH>(f, s, x, y, gather, implicit, flags), ...);
    }
};

template <bool COH = false>
__device__ __forceinline__ void load_all(double (&f)[Q], const Fld &s, int x, int y,
                                         bool gather, bool implicit, int flags) {
    LoadSeq<COH, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 21,
            22, 23, 24, 25, 26, 27, 28, 29, 30, 31, 32, 33, 34, 35,
            36>::run(f, s, x, y, gather, implicit, flags);
}

}  // namespace tlb
