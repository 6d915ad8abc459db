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

// directions d = (dx, dy): 0 left, 1 right, 2 down, 3 up, 4 down-left,
// 5 down-right, 6 up-left, 7 up-right; POPP(d) is the reverse direction
__host__ __device__ constexpr int PDX(int d) {
    return (d == 0 || d == 4 || d == 6) ? -1 : (d == 1 || d == 5 || d == 7) ? 1 : 0;
}
__host__ __device__ constexpr int PDY(int d) {
    return (d == 2 || d == 4 || d == 5) ? -1 : (d == 3 || d == 6 || d == 7) ? 1 : 0;
}
__host__ __device__ constexpr int POPP(int d) { return d < 4 ? (d ^ 1) : 11 - d; }

struct TlbPeer {
    int device = 0;
    int present[8] = {};
    double *buf[8][2] = {};              // neighbours' buffers A/B
    unsigned long long *mb[8] = {};      // neighbours' mailboxes
    void *opened[24] = {};               // IPC mappings to close (none in-process)
    unsigned long long timeout_ns = TLB_PEER_TIMEOUT_NS;
};

struct PeerLaunch {
    double *nb[8];                 // neighbours' buffers written this launch
    unsigned long long *nbmb[8];   // neighbours' mailboxes
    unsigned long long *mb;        // ours
    int present;                   // bit d: a neighbour in direction d
    long long need;                // wait until every present mailbox count >= need
    long long tag;                 // this step's number (published as tag + 1)
    int check_prev;                // our previous launch was step tag - 1
    unsigned long long timeout_ns;
    int xb, yb_lo, yb_hi;          // exchanged sides: X (both), bottom, top
    int Hx, Hy, Lx, Ly;
    unsigned nbb;                  // border blocks (the first ones)
    Rect br[4];                    // left, right (full height), bottom, top (in between)
    unsigned br_end[4];
};

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

// Wait (thread 0) until every neighbour has published step `need`; returns
// bit 0 = timeout / failed neighbour, bit 1 = step-tag mismatch.
__device__ __forceinline__ int peer_wait(const PeerLaunch &P) {
    int fail = 0;
    const unsigned long long t0 = globaltimer();
    const unsigned long long need = (unsigned long long)P.need;
    for (int d = 0; d < 8 && !(fail & 1); ++d) {
        if (!(P.present >> d & 1)) continue;
        unsigned long long v;
        while (((v = ld_acquire_sys(P.mb + d)) & TLB_MB_CTR_MASK) < need) {
            // a previous wait already failed -> a neighbour is gone; later
            // queued steps fail at once instead of waiting again
            if (ld_acquire_sys(P.mb + TLB_MB_STICKY) || globaltimer() - t0 > P.timeout_ns) {
                fail |= 1;
                break;
            }
            __nanosleep(256);
        }
        if (fail & 1) break;
        if (v & TLB_MB_POISON) {   // the neighbour failed and says so
            fail |= 1;
            break;
        }
        // step tags (Fabric.recv's check, runtime.py:151-154): a neighbour at
        // our count finished step tag-1, one ahead finished step tag
        const unsigned long long ctr = v & TLB_MB_CTR_MASK;
        const unsigned long long tag = (v >> TLB_MB_TAG_SHIFT) & TLB_MB_TAG_MASK;
        if (need > 0) {
            if (ctr == need + 1) {
                if (tag != ((unsigned long long)(P.tag + 1) & TLB_MB_TAG_MASK)) fail |= 2;
            } else if (ctr == need) {
                if (P.check_prev && tag != ((unsigned long long)P.tag & TLB_MB_TAG_MASK)) fail |= 2;
            } else {
                fail |= 2;
            }
        }
    }
    if (fail & 1) atomicExch(P.mb + TLB_MB_STICKY, 1ull);
    return fail;
}

// Debug (TLB_F_POISON_HALOS, runtime.py:288-294): NaN into every halo cell of
// f -- run by the last border block after all border blocks read the halos
// and before the step is published, i.e. before any neighbour may write
// them again.  Whatever a later step reads from a halo was stored there by
// a neighbour in between.
__device__ void poison_halos(const Fld &f) {
    const long long NY = f.Ly + 2 * f.Hy;
    const long long nxh = 2LL * f.Hx * NY, nyh = 2LL * f.Hy * f.Lx, per = nxh + nyh;
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    for (long long i = threadIdx.x; i < per * Q; i += blockDim.x) {
        const int l = (int)(i / per);
        const long long j = i % per;
        int x, y;
        if (j < nxh) {
            const int c = (int)(j / NY);
            x = c < f.Hx ? c : f.Lx + c;
            y = (int)(j % NY);
        } else {
            const long long k = j - nxh;
            const int r = (int)(k / f.Lx);
            y = r < f.Hy ? r : f.Ly + r;
            x = f.Hx + (int)(k % f.Lx);
        }
        f.base[(long long)l * f.sl + (long long)x * f.sx + (long long)y * f.sy] = nan;
    }
}

// PRIME: no arithmetic -- the border sites push their current (prv) values
// into the neighbours' prv halos (P.nb = the neighbours' prv buffers) and
// publish, as if they had just computed step tag: the halo fill before the
// first step after a (re)load.
template <bool EXACT, bool PRIME>
__global__ void __launch_bounds__(128, 4)
    k_peer_step(const __grid_constant__ SiteLaunch L, const __grid_constant__ PeerLaunch P) {
    // border blocks first (they may wait briefly for the neighbours while the
    // bulk fills the rest of the GPU), then wall frames, then the interior
    if (blockIdx.x >= P.nbb) {
        if constexpr (!PRIME) {
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
        }
        return;
    }
    // ---- border blocks: wait for every neighbour's step s-1 ----
    __shared__ int s_fail, s_last;
    if (threadIdx.x == 0) s_fail = peer_wait(P);
    __syncthreads();
    const int fail = s_fail;
    const unsigned total = P.br_end[3];
    const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = i < total && !(fail & 1);
    const unsigned ii = i < total ? i : total - 1;
    const int r = ii < P.br_end[0] ? 0 : ii < P.br_end[1] ? 1 : ii < P.br_end[2] ? 2 : 3;
    const unsigned loc = ii - (r ? P.br_end[r - 1] : 0u);
    const Rect &R = P.br[r];
    const int x = R.x0 + (int)(loc / R.ny), y = R.y0 + (int)(loc % R.ny);
    const int h = TLB_WALL_ROWS;
    double f[Q];
    if constexpr (PRIME) {
        load_inplace(f, L.src, x, y);
    } else {
        // The halos were stored by the neighbours while this grid may be
        // running: coherent L2 loads (ld.global.cg), never the read-only
        // path.  Only sites within 3 of a self-periodic or wall edge need
        // the implicit remapping -- the rest of the (tall) bands take the
        // branch-free gather of the interior.
        const bool remap_x = (L.flags & TLB_F_WRAP_X) && (x < P.Hx + h || x >= P.Hx + P.Lx - h);
        const bool remap_y = (L.flags & (TLB_F_WRAP_Y | TLB_F_CLAMP_Y)) &&
                             (y < P.Hy + h || y >= P.Hy + P.Ly - h);
        if (remap_x || remap_y)
            load_all<true>(f, L.src, x, y, true, true, L.flags);
        else
            load_plain<LD_COH>(f, L, x, y);
        unsigned bits = 0;
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
        if (active) {
            report(L.status, bits, x, y, L.step);
            store_all(f, L.dst, x, y);
        }
    }
    if (active) {
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
    if (threadIdx.x == 0) {
        if (fail & 1) report(L.status, TLB_ST_PEER_TIMEOUT, x, y, L.step);
        if (fail & 2) report(L.status, TLB_ST_PROTOCOL, x, y, L.step);
    }
    if (!PRIME && (L.flags & TLB_F_COUNT_NEG)) count_neg(L.status, f, active);
    // The last border block to finish publishes "step done" to every
    // neighbour.  Fence / counter / fence is the threadFenceReduction
    // pattern at system scope: every border block's halo reads and remote
    // stores precede its counter increment, and the last block's release
    // stores follow all of them.
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        s_last = atomicAdd(P.mb + TLB_MB_COUNTER, 1ull) == (unsigned long long)(P.nbb - 1);
    }
    __syncthreads();
    if (!s_last) return;
    if (!PRIME && (L.flags & TLB_F_POISON_HALOS)) {
        poison_halos(L.src);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        P.mb[TLB_MB_COUNTER] = 0;          // next step (next kernel) starts from 0
        __threadfence_system();
        unsigned long long v = ((unsigned long long)P.need + 1) |
                               (((unsigned long long)(P.tag + 1) & TLB_MB_TAG_MASK)
                                << TLB_MB_TAG_SHIFT);
        if (ld_acquire_sys(P.mb + TLB_MB_STICKY)) v |= TLB_MB_POISON;
        for (int d = 0; d < 8; ++d) {
            if (!(P.present >> d & 1)) continue;
            // we are that neighbour's neighbour in the reverse direction
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(P.nbmb[d] + POPP(d)),
                         "l"(v) : "memory");
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
int tlb_peer_destroy(tlb_peer_t p) {
    if (!p) return TLB_OK;
    cudaSetDevice(p->device);
    cudaDeviceSynchronize();
    for (int k = 0; k < 24; ++k)
        if (p->opened[k]) cudaIpcCloseMemHandle(p->opened[k]);
    delete p;
    return TLB_OK;
}

int tlb_peer_set_timeout(tlb_peer_t pr, double seconds) {
    if (!pr) return fail(TLB_ERR_CONTRACT, "null peer");
    if (!(seconds > 0.0)) return fail(TLB_ERR_CONTRACT, "timeout must be > 0");
    pr->timeout_ns = (unsigned long long)(seconds * 1e9);
    return TLB_OK;
}

// In-process neighbours (ranks driven by one process, on one or several
// GPUs): ptrs holds, per direction, the neighbour's buffer A, buffer B and
// mailbox as plain device pointers.  Peer access is enabled for neighbours on
// other devices.
int tlb_peer_create_local(int device, void *const *ptrs, const int *present, tlb_peer_t *out) {
    if (!ptrs || !present || !out) return fail(TLB_ERR_CONTRACT, "null argument");
    TLB_CUDA_CHECK(cudaSetDevice(device));
    TlbPeer *p = new TlbPeer();
    p->device = device;
    for (int d = 0; d < 8; ++d) {
        p->present[d] = present[d] != 0;
        if (!p->present[d]) continue;
        for (int k = 0; k < 3; ++k) {
            if (!ptrs[3 * d + k]) {
                delete p;
                return fail(TLB_ERR_CONTRACT, "peer direction %d: null pointer %d", d, k);
            }
            cudaPointerAttributes a;
            cudaError_t e = cudaPointerGetAttributes(&a, ptrs[3 * d + k]);
            if (e != cudaSuccess || a.type != cudaMemoryTypeDevice) {
                cudaGetLastError();
                delete p;
                return fail(TLB_ERR_CONTRACT, "peer direction %d: not a device pointer", d);
            }
            if (a.device != device) {
                int can = 0;
                TLB_CUDA_CHECK(cudaDeviceCanAccessPeer(&can, device, a.device));
                if (!can) {
                    delete p;
                    return fail(TLB_ERR_UNSUPPORTED, "device %d cannot access device %d", device,
                                a.device);
                }
                e = cudaDeviceEnablePeerAccess(a.device, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else if (e != cudaSuccess) {
                    delete p;
                    return fail(TLB_ERR_CUDA, "enable peer access: %s", cudaGetErrorString(e));
                }
            }
        }
        p->buf[d][0] = (double *)ptrs[3 * d];
        p->buf[d][1] = (double *)ptrs[3 * d + 1];
        p->mb[d] = (unsigned long long *)ptrs[3 * d + 2];
    }
    *out = p;
    return TLB_OK;
}

// Shared setup of a peer launch: border bands at the exchanged edges, bulk
// (interior + wall frames) over the rest.
static int peer_setup(tlb_peer_t pr, const TlbField *prv, const TlbField *nxt, int buf_index,
                      const TlbParams *p, int flags, TlbStatus *status,
                      unsigned long long *mailbox, int64_t peer_step, int64_t step_tag,
                      int check_prev, bool prime, SiteLaunch &L, PeerLaunch &P) {
    int e;
    if (!pr || !mailbox) return fail(TLB_ERR_CONTRACT, "null peer or mailbox");
    if ((e = check_stencil())) return e;
    if ((e = check_params(p))) return e;
    if (p->order != 4) return fail(TLB_ERR_UNSUPPORTED, "peer step: order 4 only");
    if (device_generic()) return fail(TLB_ERR_UNSUPPORTED, "peer step: D2Q37 kernels only");
    if (buf_index != 0 && buf_index != 1) return fail(TLB_ERR_CONTRACT, "buffer index must be 0/1");
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
    memset(&L, 0, sizeof L);
    L.src = mkfld(prv);
    L.dst = mkfld(nxt);
    L.P = mkphys(p);
    L.status = status;
    L.flags = flags;
    L.step = (int)step_tag;
    wall_rows(L, prv, flags);
    const int x0 = prv->Hx, x1 = prv->Hx + prv->Lx, y0 = prv->Hy, y1 = prv->Hy + prv->Ly;
    const int bx0 = x0 + (xb ? h : 0), bx1 = x1 - (xb ? h : 0);
    const int by0 = y0 + (yb_lo ? h : 0), by1 = y1 - (yb_hi ? h : 0);
    if (prime) {
        L.in = mkrect(0, 0, 0, 0);
        set_frames(L, nullptr, 0);
    } else {
        TlbRegion bulk = {bx0, bx1, by0, by1};
        split_region(L, bulk, prv, flags);
    }
    for (int l = 0; l < Q; ++l) {
        L.soffb[l] = 8 * ((long long)l * L.src.sl - ((long long)CX(l) * L.src.sx +
                                                      (long long)CY(l) * L.src.sy));
        L.doffb[l] = 8 * (long long)l * L.dst.sl;
    }
    L.nfb = (L.fr_end[3] + 127) / 128;
    memset(&P, 0, sizeof P);
    for (int d = 0; d < 8; ++d) {
        if (!pr->present[d]) continue;
        P.present |= 1 << d;
        P.nb[d] = pr->buf[d][buf_index];
        P.nbmb[d] = pr->mb[d];
    }
    P.mb = mailbox;
    P.need = peer_step;
    P.tag = step_tag;
    P.check_prev = check_prev;
    P.timeout_ns = pr->timeout_ns;
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
    return TLB_OK;
}

int tlb_peer_step(tlb_peer_t pr, const TlbField *prv, const TlbField *nxt, int parity,
                  const TlbParams *p, int flags, TlbStatus *status, unsigned long long *mailbox,
                  int64_t peer_step, int64_t step_tag, int check_prev, tlb_stream_t stream) {
    SiteLaunch L;
    PeerLaunch P;
    int e = peer_setup(pr, prv, nxt, parity, p, flags, status, mailbox, peer_step, step_tag,
                       check_prev, false, L, P);
    if (e) return e;
    if (prv->base == nxt->base) return fail(TLB_ERR_CONTRACT, "peer step: prv and nxt alias");
    const unsigned nb = L.nfb + (L.in.n + 127) / 128 + P.nbb;
    cudaStream_t s = (cudaStream_t)stream;
    if (p->arith == TLB_ARITH_EXACT)
        k_peer_step<true, false><<<nb, 128, 0, s>>>(L, P);
    else
        k_peer_step<false, false><<<nb, 128, 0, s>>>(L, P);
    return launch_check("peer step");
}

int tlb_peer_prime(tlb_peer_t pr, const TlbField *prv, int prv_index, const TlbParams *p,
                   TlbStatus *status, unsigned long long *mailbox, int64_t peer_step,
                   int64_t step_tag, tlb_stream_t stream) {
    SiteLaunch L;
    PeerLaunch P;
    int e = peer_setup(pr, prv, prv, prv_index, p, 0, status, mailbox, peer_step, step_tag, 0,
                       true, L, P);
    if (e) return e;
    k_peer_step<false, true><<<P.nbb, 128, 0, (cudaStream_t)stream>>>(L, P);
    return launch_check("peer prime");
}

}  // extern "C"

// ---- two steps per launch on the 1-D ring (tb2.cu, PEER) -----------------
static int tb2_peer_setup(tlb_peer_t pr, const TlbField *prv, const TlbField *nxt, int buf_index,
                          const TlbParams *p, int flags, TlbStatus *st1, TlbStatus *st2,
                          unsigned long long *mailbox, int64_t peer_step, int64_t step,
                          int check_prev, tb2::TbLaunch &T, int &sms) {
    if (!pr || !mailbox) return fail(TLB_ERR_CONTRACT, "null peer or mailbox");
    if (!pr->present[0] || !pr->present[1])
        return fail(TLB_ERR_CONTRACT, "two-step peer launch: needs left and right neighbours");
    for (int d = 2; d < 8; ++d)
        if (pr->present[d])
            return fail(TLB_ERR_UNSUPPORTED, "two-step peer launch: 1-D X ring only");
    if (buf_index != 0 && buf_index != 1) return fail(TLB_ERR_CONTRACT, "buffer index must be 0/1");
    if (prv->Hx < 6) return fail(TLB_ERR_CONTRACT, "two-step peer launch: X halo must be >= 6");
    if (prv->Lx < 12) return fail(TLB_ERR_UNSUPPORTED, "two-step peer launch: tile narrower than 12");
    if (flags & TLB_F_WRAP_X) return fail(TLB_ERR_CONTRACT, "peer step: X halos are remote");
    int e = tb2_setup(T, prv, nxt, p, flags & (TLB_F_WALL_BOT | TLB_F_WALL_TOP | TLB_F_CLAMP_Y |
                                               TLB_F_WRAP_Y | TLB_F_COUNT_NEG),
                      st1, st2, (int)step, 1, 2, sms);
    if (e) return e;
    for (int d = 0; d < 2; ++d) {
        T.pe.nb[d] = pr->buf[d][buf_index];
        T.pe.nbmb[d] = pr->mb[d];
    }
    T.pe.mb = mailbox;
    T.pe.need = peer_step;
    T.pe.tag = step;
    T.pe.check_prev = check_prev;
    T.pe.span = 2;
    T.pe.timeout_ns = pr->timeout_ns;
    T.pe.edges = 2LL * T.ns;
    T.pe.interior = T.items - T.pe.edges;
    // the work counter lives in this rank's mailbox ([10]): ranks sharing a
    // GPU run their launches concurrently and must not share it
    T.ctr = reinterpret_cast<unsigned *>(mailbox + TLB_MB_WORK);
    return TLB_OK;
}

extern "C" {

int tlb_peer_step2(tlb_peer_t pr, const TlbField *prv, const TlbField *nxt, int nxt_index,
                   const TlbParams *p, int flags, TlbStatus *status1, TlbStatus *status2,
                   unsigned long long *mailbox, int64_t peer_step, int64_t step_tag,
                   int check_prev, tlb_stream_t stream) {
    tb2::TbLaunch T;
    int sms = 0;
    int e = tb2_peer_setup(pr, prv, nxt, nxt_index, p, flags, status1, status2, mailbox,
                           peer_step, step_tag, check_prev, T, sms);
    if (e) return e;
    TLB_CUDA_CHECK(cudaMemsetAsync(T.ctr, 0, sizeof(unsigned), (cudaStream_t)stream));
    TLB_CUDA_CHECK(tb2_launch_peer(T, p->arith == TLB_ARITH_EXACT, sms, (cudaStream_t)stream));
    return TLB_OK;
}

int tlb_peer_prime2(tlb_peer_t pr, const TlbField *prv, int prv_index, const TlbParams *p,
                    TlbStatus *status, unsigned long long *mailbox, int64_t peer_step,
                    int64_t step_tag, tlb_stream_t stream) {
    tb2::TbLaunch T;
    int sms = 0;
    // any second buffer will do for the checks: the prime reads prv only
    TlbField other = *prv;
    other.base = prv->base + 1;
    int e = tb2_peer_setup(pr, prv, &other, prv_index, p, 0, status, status, mailbox, peer_step,
                           step_tag, 0, T, sms);
    if (e) return e;
    T.pe.span = 1;          // published as one step (step_tag)
    TLB_CUDA_CHECK(tb2_prime_peer(T, (cudaStream_t)stream));
    return TLB_OK;
}

}  // extern "C"
