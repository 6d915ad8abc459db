// tlb_peer.cuh -- the X-halo exchange fused into the step kernel over
// NVLink peer memory (1-D ring, one process per GPU).
//
// The border columns a rank computes at step s are exactly the halo its
// neighbours read at step s+1.  So instead of pack -> NCCL -> unpack, the
// threads that compute the 3 edge columns store their outputs twice: all 37
// into the local nxt buffer and the face-crossing ones, through CUDA-IPC-mapped
// pointers, straight into the neighbour's nxt buffer's halo columns (NVLink
// stores).  One launch per step does bulk + borders + the transfer + the
// signal: the last border block to finish publishes "step s done" into both
// neighbours' mailboxes (st.release.sys); only border blocks read our halos
// or write theirs, so the bulk need not finish first.
//
// Ordering (both directions reduce to one condition): at step s a rank's
// border blocks may (a) read its own halo, written by the neighbours during
// their step s-1, and (b) overwrite the neighbours' nxt halo, which the
// neighbours last read during their step s-1.  Border blocks therefore wait
// until both neighbours have published step s-1 (mailbox >= s).  Bulk blocks
// never wait.  Border blocks get the LOWEST block indices: in lock step the
// neighbours publish within microseconds, and a border block that waits
// holds one CTA slot while the bulk fills the rest of the GPU (placing them
// last instead leaves their latency as a tail: measured slower).  The wait
// is bounded (TLB_PEER_TIMEOUT_NS) and reports TLB_ST_PEER_TIMEOUT instead of
// hanging.
#pragma once

#define TLB_PEER_TIMEOUT_NS 5000000000ull

struct TlbPeer {
    int device = 0;
    // neighbours' buffers A/B (A = the one that is prv at even peer steps)
    double *left[2] = {nullptr, nullptr}, *right[2] = {nullptr, nullptr};
    unsigned long long *left_mb = nullptr, *right_mb = nullptr;  // their mailboxes
    void *opened[6] = {};
};

struct PeerLaunch {
    double *rleft, *rright;        // neighbours' nxt buffers (same layout as ours)
    unsigned long long *mb;        // our mailbox: [0] left done, [1] right done, [2] counter,
                                   // [3] sticky timeout flag
    unsigned long long *left_mb, *right_mb;  // the neighbours' mailboxes
    long long need;                // wait until both >= need
    int x_left0, x_right0, h;      // border bands [x_left0, +h), [x_right0, +h)
    int Lx;
    unsigned nbb;                  // border blocks (the last ones)
    Rect br[2];
    unsigned br_end[2];
};

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

template <bool EXACT>
__global__ void __launch_bounds__(128, 4)
    k_peer_step(const __grid_constant__ SiteLaunch L, const __grid_constant__ PeerLaunch P) {
    // border blocks first (they may wait briefly for the neighbours while the
    // bulk fills the rest of the GPU), then wall frames, then the interior
    if (blockIdx.x >= P.nbb) {
        const unsigned b = blockIdx.x - P.nbb;
        if (b < L.nfb) {
            const unsigned total = L.fr_end[3];
            const unsigned i = b * blockDim.x + threadIdx.x;
            const bool active = i < total;
            const unsigned ii = active ? i : total - 1;
            const int r = ii < L.fr_end[0] ? 0 : ii < L.fr_end[1] ? 1 : ii < L.fr_end[2] ? 2 : 3;
            const unsigned loc = ii - (r ? L.fr_end[r - 1] : 0u);
            const Rect &R = L.fr[r];
            site_body<K_FUSED, EXACT, 4, false, true>(L, R.x0 + (int)(loc / R.ny),
                                                      R.y0 + (int)(loc % R.ny), active);
        } else {
            const unsigned i = (b - L.nfb) * blockDim.x + threadIdx.x;
            const bool active = i < L.in.n;
            const unsigned ii = active ? i : L.in.n - 1;
            site_body<K_FUSED, EXACT, 4, false, false>(L, L.in.x0 + (int)(ii / L.in.ny),
                                                       L.in.y0 + (int)(ii % L.in.ny), active);
        }
        return;
    }
    // ---- border blocks: wait for both neighbours' step s-1 ----
    __shared__ int timed_out;
    if (threadIdx.x == 0) {
        timed_out = 0;
        const unsigned long long t0 = globaltimer();
        while (ld_acquire_sys(P.mb) < (unsigned long long)P.need ||
               ld_acquire_sys(P.mb + 1) < (unsigned long long)P.need) {
            // mb[3]: a previous wait already timed out -> the neighbour is
            // gone; later queued steps fail at once instead of 5 s each
            if (ld_acquire_sys(P.mb + 3) || globaltimer() - t0 > TLB_PEER_TIMEOUT_NS) {
                timed_out = 1;
                atomicExch(P.mb + 3, 1ull);
                break;
            }
            __nanosleep(256);
        }
    }
    __syncthreads();
    const unsigned total = P.br_end[1];
    const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = i < total && !timed_out;
    const unsigned ii = i < total ? i : total - 1;
    const int r = ii < P.br_end[0] ? 0 : 1;
    const unsigned loc = ii - (r ? P.br_end[0] : 0u);
    const Rect &R = P.br[r];
    const int x = R.x0 + (int)(loc / R.ny), y = R.y0 + (int)(loc % R.ny);
    double f[Q];
    const bool implicit = (L.flags & (TLB_F_WRAP_Y | TLB_F_CLAMP_Y)) != 0;
    load_all(f, L.src, x, y, true, implicit, L.flags);
    unsigned bits = 0;
    {
        const bool bot = y >= L.bot_lo && y < L.bot_hi;
        const bool top = y >= L.top_lo && y < L.top_hi;
#pragma unroll 1
        for (int side = 0; side < 2; ++side) {  // bottom wall, then top (kernels.py:190-203)
            if (!(side ? top : bot)) continue;
            const double Tw = side ? L.P.Ttop : L.P.Tbot;
            RegF rf{f};
            bits |= EXACT ? bc_exact<4>(rf, Tw) : bc_fast<4>(rf, Tw);
        }
        RegF rf{f};
        bits |= EXACT ? collide_exact<4>(rf, L.P) : collide_fast<4>(rf, L.P);
    }
    if (active) {
        report(L.status, bits, x, y, L.step);
        store_all(f, L.dst, x, y);
        // the neighbour's halo: our left band -> left neighbour's right halo
        // (column + Lx), our right band -> right neighbour's left halo (- Lx).
        // Only the populations its pull reads there cross the face: at halo
        // depth d those with c_x <= -d (left neighbour) or c_x >= d (right
        // neighbour) -- the face plan's 15 / 8 / 3 lines (runtime.py:94-107),
        // 26 of the 111 values of the 3 columns.  No per-thread fence: the
        // block barrier + one fence.sys before the border counter below
        // order them before the release.
        const bool left_band = x < P.x_left0 + P.h;
        const int d = left_band ? x - P.x_left0 + 1 : P.x_right0 + P.h - x;
        double *rb = left_band ? P.rleft : P.rright;
        const int rx = left_band ? x + P.Lx : x - P.Lx;
        double *q = rb + (long long)rx * L.dst.sx + (long long)y * L.dst.sy;
#pragma unroll
        for (int l = 0; l < Q; ++l) {
            if (left_band ? CX(l) <= -d : CX(l) >= d) q[(long long)l * L.dst.sl] = f[l];
        }
    }
    if (timed_out && threadIdx.x == 0) report(L.status, TLB_ST_PEER_TIMEOUT, x, y, L.step);
    if (L.flags & TLB_F_COUNT_NEG) count_neg(L.status, f, active);
    // The last border block to finish publishes "step done" to both
    // neighbours: only border blocks read our halos and write theirs, so the
    // bulk need not finish first.  Fence / counter / fence is the
    // threadFenceReduction pattern at system scope: every border block's
    // halo reads and remote stores precede its counter increment, and the
    // last block's release stores follow all of them.
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        unsigned long long *ctr = P.mb + 2;
        if (atomicAdd(ctr, 1ull) == (unsigned long long)(P.nbb - 1)) {
            *ctr = 0;                      // next step (next kernel) starts from 0
            __threadfence_system();
            const unsigned long long v = (unsigned long long)P.need + 1;
            // we are our left neighbour's RIGHT neighbour and vice versa
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(P.left_mb + 1), "l"(v)
                         : "memory");
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(P.right_mb), "l"(v)
                         : "memory");
        }
    }
}

extern "C" {

int tlb_ipc_handle(const void *ptr, char *out64, int64_t *offset) {
    // the IPC handle names the whole allocation: export its base + our offset
    using GetRange = int (*)(unsigned long long *, size_t *, unsigned long long);
    static GetRange range = nullptr;
    if (!range) {
        void *h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libcuda.so.1", RTLD_NOW);
        if (h) range = reinterpret_cast<GetRange>(dlsym(h, "cuMemGetAddressRange_v2"));
        if (!range) return fail(TLB_ERR_UNSUPPORTED, "cuMemGetAddressRange unavailable");
    }
    unsigned long long base = 0;
    size_t size = 0;
    if (range(&base, &size, (unsigned long long)ptr) != 0)
        return fail(TLB_ERR_CUDA, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t hd;
    TLB_CUDA_CHECK(cudaIpcGetMemHandle(&hd, (void *)base));
    memcpy(out64, &hd, sizeof hd);
    *offset = (int64_t)((unsigned long long)ptr - base);
    return TLB_OK;
}

int tlb_peer_create(int device, const char *handles, const int64_t *offsets, tlb_peer_t *out) {
    TLB_CUDA_CHECK(cudaSetDevice(device));
    TlbPeer *p = new TlbPeer();
    p->device = device;
    void *ptrs[6];
    for (int k = 0; k < 6; ++k) {
        cudaIpcMemHandle_t hd;
        memcpy(&hd, handles + 64 * k, sizeof hd);
        // a neighbour may appear twice (Np = 2): open each distinct handle once
        int same = -1;
        for (int j = 0; j < k; ++j)
            if (!memcmp(handles + 64 * j, handles + 64 * k, sizeof hd)) same = j;
        if (same >= 0) {
            ptrs[k] = (char *)ptrs[same] - offsets[same];
        } else {
            cudaError_t e = cudaIpcOpenMemHandle(&ptrs[k], hd, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                for (int j = 0; j < k; ++j)
                    if (p->opened[j]) cudaIpcCloseMemHandle(p->opened[j]);
                delete p;
                return fail(TLB_ERR_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
            }
            p->opened[k] = ptrs[k];
        }
        ptrs[k] = (char *)ptrs[k] + offsets[k];
    }
    p->left[0] = (double *)ptrs[0];
    p->left[1] = (double *)ptrs[1];
    p->left_mb = (unsigned long long *)ptrs[2];
    p->right[0] = (double *)ptrs[3];
    p->right[1] = (double *)ptrs[4];
    p->right_mb = (unsigned long long *)ptrs[5];
    *out = p;
    return TLB_OK;
}

int tlb_peer_destroy(tlb_peer_t p) {
    if (!p) return TLB_OK;
    cudaSetDevice(p->device);
    cudaDeviceSynchronize();
    for (int k = 0; k < 6; ++k)
        if (p->opened[k]) cudaIpcCloseMemHandle(p->opened[k]);
    delete p;
    return TLB_OK;
}

int tlb_peer_step(tlb_peer_t pr, const TlbField *prv, const TlbField *nxt, int parity,
                  const TlbParams *p, int flags, TlbStatus *status, unsigned long long *mailbox,
                  int64_t peer_step, tlb_stream_t stream) {
    int e;
    if ((e = check_stencil())) return e;
    if ((e = check_params(p))) return e;
    if (p->order != 4) return fail(TLB_ERR_UNSUPPORTED, "peer step: order 4 only");
    if (device_generic()) return fail(TLB_ERR_UNSUPPORTED, "peer step: D2Q37 kernels only");
    if (flags & (TLB_F_WRAP_X)) return fail(TLB_ERR_CONTRACT, "peer step: X halos are remote");
    const int h = TLB_WALL_ROWS;
    if (prv->Lx < 2 * h + 1) return fail(TLB_ERR_UNSUPPORTED, "peer step: tile narrower than 7");
    cudaStream_t s = (cudaStream_t)stream;
    SiteLaunch L;
    memset(&L, 0, sizeof L);
    L.src = mkfld(prv);
    L.dst = mkfld(nxt);
    L.P = mkphys(p);
    L.status = status;
    L.flags = flags;
    L.step = -1;
    wall_rows(L, prv, flags);
    TlbRegion bulk = {prv->Hx + h, prv->Hx + prv->Lx - h, prv->Hy, prv->Hy + prv->Ly};
    split_region(L, bulk, prv, flags);
    for (int l = 0; l < Q; ++l) {
        L.soffb[l] = 8 * ((long long)l * L.src.sl - ((long long)CX(l) * L.src.sx +
                                                      (long long)CY(l) * L.src.sy));
        L.doffb[l] = 8 * (long long)l * L.dst.sl;
    }
    L.nfb = (L.fr_end[3] + 127) / 128;
    PeerLaunch P;
    memset(&P, 0, sizeof P);
    P.rleft = pr->left[parity];
    P.rright = pr->right[parity];
    P.mb = mailbox;
    P.left_mb = pr->left_mb;
    P.right_mb = pr->right_mb;
    P.need = peer_step;
    P.h = h;
    P.Lx = prv->Lx;
    P.x_left0 = prv->Hx;
    P.x_right0 = prv->Hx + prv->Lx - h;
    P.br[0] = mkrect(prv->Hx, prv->Hx + h, prv->Hy, prv->Hy + prv->Ly);
    P.br[1] = mkrect(prv->Hx + prv->Lx - h, prv->Hx + prv->Lx, prv->Hy, prv->Hy + prv->Ly);
    P.br_end[0] = P.br[0].n;
    P.br_end[1] = P.br[0].n + P.br[1].n;
    P.nbb = (P.br_end[1] + 127) / 128;
    const unsigned nb = L.nfb + (L.in.n + 127) / 128 + P.nbb;
    if (p->arith == TLB_ARITH_EXACT)
        k_peer_step<true><<<nb, 128, 0, s>>>(L, P);
    else
        k_peer_step<false><<<nb, 128, 0, s>>>(L, P);
    return launch_check("peer step");
}

}  // extern "C"
