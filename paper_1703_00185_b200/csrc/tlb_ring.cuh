// tlb_ring.cuh -- halo-exchange step across GPUs (one process per GPU):
// the 1-D X ring and the 2-D grid of the reference (decompose,
// runtime.py:54-91).
//
// Replaces RankWorker.pbc_nc/pbc_c + the overlapped schedule of
// RankWorker.step (runtime.py:248-284, 378-396) for ranks on different GPUs.
// One call enqueues a whole time step with no host synchronisation:
//
//   main stream : --ev_pack--> bulk fused kernel ......................... wait ev_done
//   side stream : wait ev_pack; [2-D: pack Y faces, ncclGroup{Y}, unpack Y];
//                 pack X faces (full height: corners carry diagonal data);
//                 ncclGroup{send+,recv+,send-,recv-}; unpack X halos;
//                 fused kernel on the frame bands; record ev_done
//
// The side stream has the highest priority, so the NCCL kernel and the
// border blocks are dispatched into SM slots as bulk CTAs retire: the
// exchange and the borders overlap the bulk columns.  NCCL is resolved at
// run time (dlopen "libnccl.so.2"): in a PyTorch process this is the NCCL
// torch already loaded, so only one NCCL lives in the process.
#pragma once
#include <dlfcn.h>

#include <nccl.h>

namespace tlbring {

struct Nccl {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetVersion)(int *) = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
};

static Nccl &nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n.why = std::string("dlopen libnccl.so.2: ") + dlerror();
            return;
        }
#define TLB_SYM(f)                                                   \
    n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, "nccl" #f));      \
    if (!n.f) {                                                      \
        n.why = "libnccl.so.2 lacks nccl" #f;                        \
        return;                                                      \
    }
        TLB_SYM(GetVersion) TLB_SYM(GetUniqueId) TLB_SYM(CommInitRank) TLB_SYM(CommDestroy)
        TLB_SYM(CommAbort) TLB_SYM(Send) TLB_SYM(Recv) TLB_SYM(GroupStart) TLB_SYM(GroupEnd)
        TLB_SYM(GetErrorString) TLB_SYM(CommGetAsyncError)
#undef TLB_SYM
        n.ok = true;
    });
    return n;
}

}  // namespace tlbring

struct TlbRing {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0, left = 0, right = 0, device = 0;
    int up = -1, down = -1;   // 2-D tiling: Y neighbours (-1: wall side)
    double *ybuf = nullptr;   // 4 Y payloads: send up, send down, from down, from up
    cudaStream_t side = nullptr;
    cudaEvent_t ev_pack = nullptr, ev_done = nullptr;
};

#define TLB_NCCL_CHECK(expr)                                                              \
    do {                                                                                  \
        ncclResult_t _r = (expr);                                                         \
        if (_r != ncclSuccess)                                                            \
            return fail(TLB_ERR_CUDA, "%s: %s", #expr, tlbring::nccl().GetErrorString(_r)); \
    } while (0)

// Payload layout per face: the face-plan lines, then one double holding the
// sender's step number (the step tag of Fabric.send/recv, runtime.py:141-160):
// a receiver at another step flags TLB_ST_PROTOCOL instead of consuming
// halos of the wrong step.
// pack / unpack both X faces in one launch each (stride = lines * NY + 1)
__global__ void k_pack2(Fld f, FaceLines tp, FaceLines tm, int ymode, double *buf, int stride,
                        double tag) {
    const int NY = f.Ly + 2 * f.Hy;
    const int k = blockIdx.y;
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    if (k == 0 && y == 0) {
        buf[stride - 1] = tag;
        buf[2 * stride - 1] = tag;
    }
    if (y >= NY) return;
    const bool plus = k < tp.n;
    const int kk = plus ? k : k - tp.n;
    if (!plus && kk >= tm.n) return;
    const int l = plus ? tp.l[kk] : tm.l[kk];
    const int d = plus ? tp.d[kk] : tm.d[kk];
    const int col = plus ? f.Hx + f.Lx - d : f.Hx + d - 1;
    const int ys = ysrc_mode(y, f, ymode);
    double *out = buf + (plus ? 0 : stride);
    out[(long long)kk * NY + y] =
        f.base[(long long)l * f.sl + (long long)col * f.sx + (long long)ys * f.sy];
}

__device__ __forceinline__ void check_tags(const double *a, const double *b, double expect,
                                           TlbStatus *st, int step) {
    if (st && expect >= 0.0 && (a[0] != expect || b[0] != expect))
        report(st, TLB_ST_PROTOCOL, -1, -1, step);
}

__global__ void k_unpack2(Fld f, FaceLines tp, FaceLines tm, const double *buf, int stride,
                          double expect, TlbStatus *st) {
    const int NY = f.Ly + 2 * f.Hy;
    const int k = blockIdx.y;
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    if (k == 0 && y == 0) check_tags(buf + stride - 1, buf + 2 * stride - 1, expect, st, (int)expect);
    if (y >= NY) return;
    const bool plus = k < tp.n;  // arrived travelling +x: from the left -> low-x halo
    const int kk = plus ? k : k - tp.n;
    if (!plus && kk >= tm.n) return;
    const int l = plus ? tp.l[kk] : tm.l[kk];
    const int d = plus ? tp.d[kk] : tm.d[kk];
    const int col = plus ? f.Hx - d : f.Hx + f.Lx - 1 + d;
    const double *in = buf + (plus ? 0 : stride);
    f.base[(long long)l * f.sl + (long long)col * f.sx + (long long)y * f.sy] =
        in[(long long)kk * NY + y];
}

__global__ void k_tags_put(double *a, double *b, double tag) {
    if (a) a[0] = tag;
    if (b) b[0] = tag;
}

__global__ void k_tags_check(const double *a, const double *b, double expect, TlbStatus *st) {
    if (st && expect >= 0.0 && ((a && a[0] != expect) || (b && b[0] != expect)))
        report(st, TLB_ST_PROTOCOL, -1, -1, (int)expect);
}

static int ring_stride(const TlbField *f) { return (int)tlb_face_payload_len(f) + 1; }

static int ring_pack(const TlbField *f, int ymode, double *sbuf, double tag, cudaStream_t s) {
    FaceLines tp = face_lines(1, 0), tm = face_lines(-1, 0);
    const int NY = f->Ly + 2 * f->Hy;
    dim3 grid((NY + 127) / 128, tp.n + tm.n);
    k_pack2<<<grid, 128, 0, s>>>(mkfld(f), tp, tm, ymode, sbuf, ring_stride(f), tag);
    return launch_check("ring pack");
}

static int ring_unpack(const TlbField *f, const double *rbuf, double expect, TlbStatus *st,
                       cudaStream_t s) {
    FaceLines tp = face_lines(1, 0), tm = face_lines(-1, 0);
    const int NY = f->Ly + 2 * f->Hy;
    dim3 grid((NY + 127) / 128, tp.n + tm.n);
    k_unpack2<<<grid, 128, 0, s>>>(mkfld(f), tp, tm, rbuf, ring_stride(f), expect, st);
    return launch_check("ring unpack");
}

// Y faces (pbc_nc, runtime.py:248-267): rows of physical columns travel up
// and down; the group order pairs each send with the matching receive even
// when up == down (two ranks on a periodic Y ring).  Each payload carries
// the step tag after its lines (stride n + 1).
static int ring_exchange_y(TlbRing *r, const TlbField *f, double tag, TlbStatus *st,
                           cudaStream_t s) {
    auto &N = tlbring::nccl();
    const size_t n = (size_t)tlb_face_payload_len_y(f), m = n + 1;
    double *s_up = r->ybuf, *s_dn = r->ybuf + m, *r_dn = r->ybuf + 2 * m, *r_up = r->ybuf + 3 * m;
    int e;
    if (r->up >= 0 && (e = tlb_pack_y(f, 1, s_up, s))) return e;
    if (r->down >= 0 && (e = tlb_pack_y(f, -1, s_dn, s))) return e;
    k_tags_put<<<1, 1, 0, s>>>(r->up >= 0 ? s_up + n : nullptr, r->down >= 0 ? s_dn + n : nullptr,
                               tag);
    TLB_NCCL_CHECK(N.GroupStart());
    if (r->up >= 0) TLB_NCCL_CHECK(N.Send(s_up, m, ncclFloat64, r->up, r->comm, s));
    if (r->down >= 0) TLB_NCCL_CHECK(N.Recv(r_dn, m, ncclFloat64, r->down, r->comm, s));
    if (r->down >= 0) TLB_NCCL_CHECK(N.Send(s_dn, m, ncclFloat64, r->down, r->comm, s));
    if (r->up >= 0) TLB_NCCL_CHECK(N.Recv(r_up, m, ncclFloat64, r->up, r->comm, s));
    TLB_NCCL_CHECK(N.GroupEnd());
    k_tags_check<<<1, 1, 0, s>>>(r->down >= 0 ? r_dn + n : nullptr, r->up >= 0 ? r_up + n : nullptr,
                                 tag, st);
    if (r->down >= 0 && (e = tlb_unpack_y(f, 1, r_dn, s))) return e;
    if (r->up >= 0 && (e = tlb_unpack_y(f, -1, r_up, s))) return e;
    return TLB_OK;
}

static int ring_exchange(TlbRing *r, size_t stride, const double *sbuf, double *rbuf,
                         cudaStream_t s) {
    auto &N = tlbring::nccl();
    // data travelling +x goes to the right neighbour and arrives from the left
    TLB_NCCL_CHECK(N.GroupStart());
    TLB_NCCL_CHECK(N.Send(sbuf, stride, ncclFloat64, r->right, r->comm, s));
    TLB_NCCL_CHECK(N.Recv(rbuf, stride, ncclFloat64, r->left, r->comm, s));
    TLB_NCCL_CHECK(N.Send(sbuf + stride, stride, ncclFloat64, r->left, r->comm, s));
    TLB_NCCL_CHECK(N.Recv(rbuf + stride, stride, ncclFloat64, r->right, r->comm, s));
    TLB_NCCL_CHECK(N.GroupEnd());
    return TLB_OK;
}

extern "C" {

int tlb_nccl_version(int *version) {
    auto &N = tlbring::nccl();
    if (!N.ok) return fail(TLB_ERR_UNSUPPORTED, "%s", N.why.c_str());
    TLB_NCCL_CHECK(N.GetVersion(version));
    return TLB_OK;
}

int tlb_nccl_unique_id(char *out128) {
    auto &N = tlbring::nccl();
    if (!N.ok) return fail(TLB_ERR_UNSUPPORTED, "%s", N.why.c_str());
    ncclUniqueId id;
    TLB_NCCL_CHECK(N.GetUniqueId(&id));
    memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
    return TLB_OK;
}

int tlb_ring_create(const char *uid128, int nranks, int rank, int device, tlb_ring_t *out) {
    auto &N = tlbring::nccl();
    if (!N.ok) return fail(TLB_ERR_UNSUPPORTED, "%s", N.why.c_str());
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(TLB_ERR_CONTRACT, "bad rank");
    TLB_CUDA_CHECK(cudaSetDevice(device));
    ncclUniqueId id;
    memcpy(id.internal, uid128, NCCL_UNIQUE_ID_BYTES);
    TlbRing *r = new TlbRing();
    r->nranks = nranks;
    r->rank = rank;
    r->left = (rank - 1 + nranks) % nranks;   // runtime.py:76-77
    r->right = (rank + 1) % nranks;
    r->device = device;
    ncclResult_t res = N.CommInitRank(&r->comm, nranks, id, rank);
    if (res != ncclSuccess) {
        delete r;
        return fail(TLB_ERR_CUDA, "ncclCommInitRank: %s", N.GetErrorString(res));
    }
    int lo = 0, hi = 0;
    TLB_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    TLB_CUDA_CHECK(cudaStreamCreateWithPriority(&r->side, cudaStreamNonBlocking, hi));
    TLB_CUDA_CHECK(cudaEventCreateWithFlags(&r->ev_pack, cudaEventDisableTiming));
    TLB_CUDA_CHECK(cudaEventCreateWithFlags(&r->ev_done, cudaEventDisableTiming));
    *out = r;
    return TLB_OK;
}

int tlb_ring_destroy(tlb_ring_t r) {
    if (!r) return TLB_OK;
    auto &N = tlbring::nccl();
    cudaSetDevice(r->device);
    if (r->comm && r->side) cudaStreamSynchronize(r->side);
    if (r->comm && N.ok) N.CommDestroy(r->comm);
    if (r->ev_pack) cudaEventDestroy(r->ev_pack);
    if (r->ev_done) cudaEventDestroy(r->ev_done);
    if (r->side) cudaStreamDestroy(r->side);
    delete r;
    return TLB_OK;
}

int tlb_ring_async_error(tlb_ring_t r, int *nccl_result) {
    if (!r || !r->comm) return fail(TLB_ERR_CONTRACT, "null ring");
    ncclResult_t res = ncclSuccess;
    TLB_NCCL_CHECK(tlbring::nccl().CommGetAsyncError(r->comm, &res));
    *nccl_result = (int)res;
    return TLB_OK;
}

// Abort the communicator (a stalled or failed peer): outstanding NCCL
// kernels are released so the process can report the failure and exit.
int tlb_ring_abort(tlb_ring_t r) {
    if (!r || !r->comm) return TLB_OK;
    auto &N = tlbring::nccl();
    if (N.ok) N.CommAbort(r->comm);
    r->comm = nullptr;
    return TLB_OK;
}

int tlb_ring_set_neighbors(tlb_ring_t r, int left, int right, int up, int down, double *ybuf) {
    if (!r) return fail(TLB_ERR_CONTRACT, "null ring");
    const int n = r->nranks;
    if (left < 0 || left >= n || right < 0 || right >= n || up >= n || down >= n)
        return fail(TLB_ERR_CONTRACT, "neighbour rank out of range");
    if ((up >= 0 || down >= 0) && !ybuf)
        return fail(TLB_ERR_CONTRACT, "Y neighbours need a Y payload buffer");
    r->left = left;
    r->right = right;
    r->up = up < 0 ? -1 : up;
    r->down = down < 0 ? -1 : down;
    r->ybuf = ybuf;
    return TLB_OK;
}

int tlb_ring_exchange(tlb_ring_t r, const TlbField *f, int ymode, double *sbuf, double *rbuf,
                      tlb_stream_t stream) {
    cudaStream_t s = (cudaStream_t)stream;
    int e;
    if ((r->up >= 0 || r->down >= 0) && (e = ring_exchange_y(r, f, -1.0, nullptr, s))) return e;
    if ((e = ring_pack(f, ymode, sbuf, -1.0, s))) return e;
    if ((e = ring_exchange(r, (size_t)ring_stride(f), sbuf, rbuf, s))) return e;
    return ring_unpack(f, rbuf, -1.0, nullptr, s);
}

int tlb_ring_step(tlb_ring_t r, const TlbField *prv, const TlbField *nxt, const TlbParams *p,
                  int flags, TlbStatus *status, double *sbuf, double *rbuf,
                  void *ev_bulk0, void *ev_bulk1, int64_t step_tag, tlb_stream_t stream) {
    int e;
    if ((e = check_stencil())) return e;
    if ((e = check_params(p))) return e;
    if (flags & TLB_F_WRAP_X)
        return fail(TLB_ERR_CONTRACT, "ring step: X halos come from the neighbours");
    cudaStream_t s = (cudaStream_t)stream;
    const int h = TLB_WALL_ROWS;
    const bool cb = (flags & TLB_F_CLAMP_BOT) != 0, ct = (flags & TLB_F_CLAMP_TOP) != 0;
    const int ymode = (cb && ct) ? 1 : (flags & TLB_F_WRAP_Y) ? 2 : cb ? 3 : ct ? 4 : 0;
    const bool has_y = r->up >= 0 || r->down >= 0;
    // Y sides that need the exchange (not walls, not periodic self-wrap)
    const bool ex_bot = has_y && r->down >= 0, ex_top = has_y && r->up >= 0;
    // 1. everything that reads prv's faces waits for prv on the side stream
    TLB_CUDA_CHECK(cudaEventRecord(r->ev_pack, s));
    TLB_CUDA_CHECK(cudaStreamWaitEvent(r->side, r->ev_pack, 0));
    // 2. Y faces first (2-D), then X faces carrying the Y halo rows
    const double tag = (double)step_tag;
    if (has_y && (e = ring_exchange_y(r, prv, tag, status, r->side))) return e;
    if ((e = ring_pack(prv, ymode, sbuf, tag, r->side))) return e;
    if ((e = ring_exchange(r, (size_t)ring_stride(prv), sbuf, rbuf, r->side))) return e;
    // 3. bulk on the main stream, concurrent with the exchanges: all columns
    //    >= 3 from the X edges, all rows not within 3 of an exchanged Y edge
    if (ev_bulk0) TLB_CUDA_CHECK(cudaEventRecord((cudaEvent_t)ev_bulk0, s));
    const int by0 = prv->Hy + (ex_bot ? h : 0), by1 = prv->Hy + prv->Ly - (ex_top ? h : 0);
    if (prv->Lx > 2 * h && by1 > by0) {
        TlbRegion bulk = {prv->Hx + h, prv->Hx + prv->Lx - h, by0, by1};
        if ((e = tlb_fused(prv, nxt, bulk, p, flags, status, s))) return e;
    }
    if (ev_bulk1) TLB_CUDA_CHECK(cudaEventRecord((cudaEvent_t)ev_bulk1, s));
    // 4. halos in, then the frame bands (one launch) on the side stream
    if ((e = ring_unpack(prv, rbuf, tag, status, r->side))) return e;
    {
        SiteLaunch L;
        memset(&L, 0, sizeof L);
        L.src = mkfld(prv);
        L.dst = mkfld(nxt);
        L.P = mkphys(p);
        L.status = status;
        L.flags = flags;
        L.step = -1;
        wall_rows(L, prv, flags);
        L.in = mkrect(0, 0, 0, 0);
        const int x0 = prv->Hx, x1 = prv->Hx + prv->Lx, y0 = prv->Hy, y1 = prv->Hy + prv->Ly;
        Rect rs[4];
        int nr = 0;
        if (prv->Lx > 2 * h) {
            rs[nr++] = mkrect(x0, x0 + h, y0, y1);
            rs[nr++] = mkrect(x1 - h, x1, y0, y1);
            if (by1 > by0) {
                if (ex_bot) rs[nr++] = mkrect(x0 + h, x1 - h, y0, by0);
                if (ex_top) rs[nr++] = mkrect(x0 + h, x1 - h, by1, y1);
            } else {
                rs[nr++] = mkrect(x0 + h, x1 - h, y0, y1);
            }
        } else {
            rs[nr++] = mkrect(x0, x1, y0, y1);
        }
        set_frames(L, rs, nr);
        if ((e = launch_site<K_FUSED, false>(L, p->arith == TLB_ARITH_EXACT, p->order, r->side,
                                             "ring frames")))
            return e;
    }
    // 5. join
    TLB_CUDA_CHECK(cudaEventRecord(r->ev_done, r->side));
    TLB_CUDA_CHECK(cudaStreamWaitEvent(s, r->ev_done, 0));
    return TLB_OK;
}

}  // extern "C"
