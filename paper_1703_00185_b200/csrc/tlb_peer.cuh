// tlb_peer.cuh -- the halo exchange fused into the step kernel over NVLink
// peer memory (one process per GPU; 1-D ring or 2-D rank grid).
//
// The border sites a rank computes at step s are exactly the halo its
// neighbours read at step s+1.  So instead of pack -> NCCL -> unpack, the
// threads that compute the 3-wide border bands store their outputs twice:
// all 37 into the local nxt buffer and the face-crossing ones, through
// CUDA-IPC-mapped pointers, straight into the neighbours' nxt halos (NVLink
// stores).  On a 2-D grid a corner site also stores into the diagonal
// neighbour's corner halo, so no Y-before-X ordering is needed: NVSwitch
// reaches all 8 neighbours in one hop.  One launch per step does bulk +
// borders + transfer + signal: the last border block to finish publishes
// "step s done" into every neighbour's mailbox (st.release.sys); only border
// blocks read our halos or write theirs, so the bulk need not finish first.
//
// Ordering: at step s a rank's border blocks may (a) read its own halos,
// written by the neighbours during their step s-1, and (b) overwrite the
// neighbours' nxt halos, which the neighbours last read during their step
// s-1.  Border blocks therefore wait until every neighbour has published
// step s-1 (mailbox >= s).  Bulk blocks never wait.  Border blocks get the
// LOWEST block indices: in lock step the neighbours publish within
// microseconds, and a waiting border block holds one CTA slot while the bulk
// fills the rest of the GPU (placing them last leaves their latency as a
// tail: measured slower).  The wait is bounded (TLB_PEER_TIMEOUT_NS); an
// expiry flags TLB_ST_PEER_TIMEOUT and is sticky (later queued steps fail at
// once instead of waiting again).
#pragma once

#define TLB_PEER_TIMEOUT_NS 5000000000ull

// directions d = (dx, dy): 0 left, 1 right, 2 down, 3 up, 4 down-left,
// 5 down-right, 6 up-left, 7 up-right; POPP(d) is the reverse direction
__host__ __device__ constexpr int PDX(int d) {
    return (d == 0 || d == 4 || d == 6) ? -1 : (d == 1 || d == 5 || d == 7) ? 1 : 0;
}
__host__ __device__ constexpr int PDY(int d) {
    return (d == 2 || d == 4 || d == 5) ? -1 : (d == 3 || d == 6 || d == 7) ? 1 : 0;
}
__host__ __device__ constexpr int POPP(int d) { return d < 4 ? (d ^ 1) : 11 - d; }

// mailbox layout (u64): [0..7] step published by the neighbour in direction
// d, [8] border-block counter, [9] sticky timeout flag
#define TLB_MB_COUNTER 8
#define TLB_MB_STICKY 9

struct TlbPeer {
    int device = 0;
    int present[8] = {};
    double *buf[8][2] = {};              // neighbours' buffers A/B
    unsigned long long *mb[8] = {};      // neighbours' mailboxes
    void *opened[24] = {};
};

struct PeerLaunch {
    double *nb[8];                 // neighbours' nxt buffers (same layout as ours)
    unsigned long long *nbmb[8];   // neighbours' mailboxes
    unsigned long long *mb;        // ours
    int present;                   // bit d: a neighbour in direction d
    long long need;                // wait until every present mailbox slot >= need
    int xb, yb_lo, yb_hi;          // exchanged sides: X (both), bottom, top
    int Hx, Hy, Lx, Ly;
    unsigned nbb;                  // border blocks (the first ones)
    Rect br[4];                    // left, right (full height), bottom, top (in between)
    unsigned br_end[4];
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

// Store the populations of f that cross into direction d: at halo depth
// (ddx, ddy) those with c_x <= -ddx (left) / >= ddx (right) and c_y <= -ddy
// (down) / >= ddy (up) -- the face plans of runtime.py:94-107 and, at the
// corners, their intersections.  Our site (x, y) is (x - dx Lx, y - dy Ly)
// in the neighbour's frame.
template <int d>
__device__ __forceinline__ void peer_put(const PeerLaunch &P, const Fld &D, const double (&f)[Q],
                                         int x, int y, int ddx, int ddy) {
    if (!(P.present >> d & 1)) return;
    double *q = P.nb[d] + (long long)(x - PDX(d) * P.Lx) * D.sx +
                (long long)(y - PDY(d) * P.Ly) * D.sy;
#pragma unroll
    for (int l = 0; l < Q; ++l) {
        const bool okx = PDX(d) < 0 ? CX(l) <= -ddx : PDX(d) > 0 ? CX(l) >= ddx : true;
        const bool oky = PDY(d) < 0 ? CY(l) <= -ddy : PDY(d) > 0 ? CY(l) >= ddy : true;
        if (okx && oky) q[(long long)l * D.sl] = f[l];
    }
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
    // ---- border blocks: wait for every neighbour's step s-1 ----
    __shared__ int timed_out;
    if (threadIdx.x == 0) {
        int late = 0;
        const unsigned long long t0 = globaltimer();
        for (int d = 0; d < 8 && !late; ++d) {
            if (!(P.present >> d & 1)) continue;
            while (ld_acquire_sys(P.mb + d) < (unsigned long long)P.need) {
                // a previous wait already timed out -> a neighbour is gone;
                // later queued steps fail at once instead of 5 s each
                if (ld_acquire_sys(P.mb + TLB_MB_STICKY) ||
                    globaltimer() - t0 > TLB_PEER_TIMEOUT_NS) {
                    late = 1;
                    atomicExch(P.mb + TLB_MB_STICKY, 1ull);
                    break;
                }
                __nanosleep(256);
            }
        }
        timed_out = late;
    }
    __syncthreads();
    const unsigned total = P.br_end[3];
    const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = i < total && !timed_out;
    const unsigned ii = i < total ? i : total - 1;
    const int r = ii < P.br_end[0] ? 0 : ii < P.br_end[1] ? 1 : ii < P.br_end[2] ? 2 : 3;
    const unsigned loc = ii - (r ? P.br_end[r - 1] : 0u);
    const Rect &R = P.br[r];
    const int x = R.x0 + (int)(loc / R.ny), y = R.y0 + (int)(loc % R.ny);
    double f[Q];
    // the halos are in memory (neighbours' stores); only sites within 3 of a
    // self-periodic or wall edge need the implicit remapping -- the rest of
    // the (tall) bands take the branch-free gather of the interior
    const int h = TLB_WALL_ROWS;
    const bool remap_x = (L.flags & TLB_F_WRAP_X) && (x < P.Hx + h || x >= P.Hx + P.Lx - h);
    const bool remap_y = (L.flags & (TLB_F_WRAP_Y | TLB_F_CLAMP_Y)) &&
                         (y < P.Hy + h || y >= P.Hy + P.Ly - h);
    if (remap_x || remap_y)
        load_all(f, L.src, x, y, true, true, L.flags);
    else
        load_plain<false>(f, L, x, y);
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
        // depth of this site inside each exchanged band (0 = not in it).  No
        // per-thread fence: the block barrier + one fence.sys before the
        // border counter below order these stores before the release.
        const int dl = P.xb && x < P.Hx + h ? x - P.Hx + 1 : 0;
        const int dr = P.xb && x >= P.Hx + P.Lx - h ? P.Hx + P.Lx - x : 0;
        const int db = P.yb_lo && y < P.Hy + h ? y - P.Hy + 1 : 0;
        const int dt = P.yb_hi && y >= P.Hy + P.Ly - h ? P.Hy + P.Ly - y : 0;
        if (dl) peer_put<0>(P, L.dst, f, x, y, dl, 0);
        if (dr) peer_put<1>(P, L.dst, f, x, y, dr, 0);
        if (db) peer_put<2>(P, L.dst, f, x, y, 0, db);
        if (dt) peer_put<3>(P, L.dst, f, x, y, 0, dt);
        if (dl && db) peer_put<4>(P, L.dst, f, x, y, dl, db);
        if (dr && db) peer_put<5>(P, L.dst, f, x, y, dr, db);
        if (dl && dt) peer_put<6>(P, L.dst, f, x, y, dl, dt);
        if (dr && dt) peer_put<7>(P, L.dst, f, x, y, dr, dt);
    }
    if (timed_out && threadIdx.x == 0) report(L.status, TLB_ST_PEER_TIMEOUT, x, y, L.step);
    if (L.flags & TLB_F_COUNT_NEG) count_neg(L.status, f, active);
    // The last border block to finish publishes "step done" to every
    // neighbour.  Fence / counter / fence is the threadFenceReduction
    // pattern at system scope: every border block's halo reads and remote
    // stores precede its counter increment, and the last block's release
    // stores follow all of them.
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        unsigned long long *ctr = P.mb + TLB_MB_COUNTER;
        if (atomicAdd(ctr, 1ull) == (unsigned long long)(P.nbb - 1)) {
            *ctr = 0;                      // next step (next kernel) starts from 0
            __threadfence_system();
            const unsigned long long v = (unsigned long long)P.need + 1;
            for (int d = 0; d < 8; ++d) {
                if (!(P.present >> d & 1)) continue;
                // we are that neighbour's neighbour in the reverse direction
                asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(P.nbmb[d] + POPP(d)),
                             "l"(v) : "memory");
            }
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

int tlb_peer_create2(int device, const char *handles, const int64_t *offsets,
                     const int *present, tlb_peer_t *out) {
    TLB_CUDA_CHECK(cudaSetDevice(device));
    TlbPeer *p = new TlbPeer();
    p->device = device;
    void *ptrs[24] = {};
    for (int k = 0; k < 24; ++k) {
        if (!present[k / 3]) continue;
        cudaIpcMemHandle_t hd;
        memcpy(&hd, handles + 64 * k, sizeof hd);
        // a neighbour can sit in several directions: open each handle once
        int same = -1;
        for (int j = 0; j < k; ++j)
            if (present[j / 3] && !memcmp(handles + 64 * j, handles + 64 * k, sizeof hd))
                same = j;
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
    for (int d = 0; d < 8; ++d) {
        p->present[d] = present[d] != 0;
        p->buf[d][0] = (double *)ptrs[3 * d];
        p->buf[d][1] = (double *)ptrs[3 * d + 1];
        p->mb[d] = (unsigned long long *)ptrs[3 * d + 2];
    }
    *out = p;
    return TLB_OK;
}

// 1-D ring: handles/offsets = left A, left B, left mailbox, right A, right B,
// right mailbox
int tlb_peer_create(int device, const char *handles, const int64_t *offsets, tlb_peer_t *out) {
    char h[24 * 64] = {};
    int64_t o[24] = {};
    const int present[8] = {1, 1, 0, 0, 0, 0, 0, 0};
    memcpy(h, handles, 6 * 64);
    memcpy(o, offsets, 6 * sizeof(int64_t));
    return tlb_peer_create2(device, h, o, present, out);
}

int tlb_peer_destroy(tlb_peer_t p) {
    if (!p) return TLB_OK;
    cudaSetDevice(p->device);
    cudaDeviceSynchronize();
    for (int k = 0; k < 24; ++k)
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
    const int h = TLB_WALL_ROWS;
    const bool xb = pr->present[0] || pr->present[1];
    const bool yb_lo = pr->present[2], yb_hi = pr->present[3];
    if (!xb && !yb_lo && !yb_hi) return fail(TLB_ERR_CONTRACT, "peer step: no neighbours");
    if (xb && (flags & TLB_F_WRAP_X))
        return fail(TLB_ERR_CONTRACT, "peer step: X halos are remote");
    if ((yb_lo || yb_hi) && (flags & TLB_F_WRAP_Y))
        return fail(TLB_ERR_CONTRACT, "peer step: Y halos are remote");
    if (xb && prv->Lx < 2 * h + 1)
        return fail(TLB_ERR_UNSUPPORTED, "peer step: tile narrower than 7");
    if ((yb_lo || yb_hi) && prv->Ly < 2 * h + 1)
        return fail(TLB_ERR_UNSUPPORTED, "peer step: tile lower than 7");
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
    const int x0 = prv->Hx, x1 = prv->Hx + prv->Lx, y0 = prv->Hy, y1 = prv->Hy + prv->Ly;
    const int bx0 = x0 + (xb ? h : 0), bx1 = x1 - (xb ? h : 0);
    const int by0 = y0 + (yb_lo ? h : 0), by1 = y1 - (yb_hi ? h : 0);
    TlbRegion bulk = {bx0, bx1, by0, by1};
    split_region(L, bulk, prv, flags);
    for (int l = 0; l < Q; ++l) {
        L.soffb[l] = 8 * ((long long)l * L.src.sl - ((long long)CX(l) * L.src.sx +
                                                      (long long)CY(l) * L.src.sy));
        L.doffb[l] = 8 * (long long)l * L.dst.sl;
    }
    L.nfb = (L.fr_end[3] + 127) / 128;
    PeerLaunch P;
    memset(&P, 0, sizeof P);
    for (int d = 0; d < 8; ++d) {
        if (!pr->present[d]) continue;
        P.present |= 1 << d;
        P.nb[d] = pr->buf[d][parity];
        P.nbmb[d] = pr->mb[d];
    }
    P.mb = mailbox;
    P.need = peer_step;
    P.xb = xb;
    P.yb_lo = yb_lo;
    P.yb_hi = yb_hi;
    P.Hx = prv->Hx;
    P.Hy = prv->Hy;
    P.Lx = prv->Lx;
    P.Ly = prv->Ly;
    // border bands: left / right columns over the full height, then bottom /
    // top rows between them
    const Rect none = mkrect(0, 0, 0, 0);
    P.br[0] = xb ? mkrect(x0, x0 + h, y0, y1) : none;
    P.br[1] = xb ? mkrect(x1 - h, x1, y0, y1) : none;
    P.br[2] = yb_lo ? mkrect(bx0, bx1, y0, y0 + h) : none;
    P.br[3] = yb_hi ? mkrect(bx0, bx1, y1 - h, y1) : none;
    unsigned acc = 0;
    for (int k = 0; k < 4; ++k) {
        acc += P.br[k].n;
        P.br_end[k] = acc;
    }
    P.nbb = (acc + 127) / 128;
    const unsigned nb = L.nfb + (L.in.n + 127) / 128 + P.nbb;
    if (p->arith == TLB_ARITH_EXACT)
        k_peer_step<true><<<nb, 128, 0, s>>>(L, P);
    else
        k_peer_step<false><<<nb, 128, 0, s>>>(L, P);
    return launch_check("peer step");
}

}  // extern "C"
