// tlb_ring.cuh -- 1-D X ring step across GPUs (one process per GPU).
//
// Replaces RankWorker.pbc_c + the overlapped schedule of RankWorker.step
// (runtime.py:269-284, 378-396) for ranks on different GPUs.  One call
// enqueues a whole time step with no host synchronisation:
//
//   main stream : pack both X faces --ev_pack--> bulk fused kernel  ...wait ev_done
//   side stream : wait ev_pack; ncclGroup{send+,recv+,send-,recv-};
//                 unpack both halos; fused kernel on the 3+3 border columns;
//                 record ev_done
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
        TLB_SYM(GetErrorString)
#undef TLB_SYM
        n.ok = true;
    });
    return n;
}

}  // namespace tlbring

struct TlbRing {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0, left = 0, right = 0, device = 0;
    cudaStream_t side = nullptr;
    cudaEvent_t ev_pack = nullptr, ev_done = nullptr;
};

#define TLB_NCCL_CHECK(expr)                                                              \
    do {                                                                                  \
        ncclResult_t _r = (expr);                                                         \
        if (_r != ncclSuccess)                                                            \
            return fail(TLB_ERR_CUDA, "%s: %s", #expr, tlbring::nccl().GetErrorString(_r)); \
    } while (0)

// pack / unpack both X faces in one launch each
__global__ void k_pack2(Fld f, FaceLines tp, FaceLines tm, int ymode, double *buf, int n_per) {
    const int NY = f.Ly + 2 * f.Hy;
    const int k = blockIdx.y;
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= NY) return;
    const bool plus = k < tp.n;
    const int kk = plus ? k : k - tp.n;
    if (!plus && kk >= tm.n) return;
    const int l = plus ? tp.l[kk] : tm.l[kk];
    const int d = plus ? tp.d[kk] : tm.d[kk];
    const int col = plus ? f.Hx + f.Lx - d : f.Hx + d - 1;
    const int ys = ysrc_mode(y, f, ymode);
    double *out = buf + (plus ? 0 : n_per);
    out[(long long)kk * NY + y] =
        f.base[(long long)l * f.sl + (long long)col * f.sx + (long long)ys * f.sy];
}

__global__ void k_unpack2(Fld f, FaceLines tp, FaceLines tm, const double *buf, int n_per) {
    const int NY = f.Ly + 2 * f.Hy;
    const int k = blockIdx.y;
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= NY) return;
    const bool plus = k < tp.n;  // arrived travelling +x: from the left -> low-x halo
    const int kk = plus ? k : k - tp.n;
    if (!plus && kk >= tm.n) return;
    const int l = plus ? tp.l[kk] : tm.l[kk];
    const int d = plus ? tp.d[kk] : tm.d[kk];
    const int col = plus ? f.Hx - d : f.Hx + f.Lx - 1 + d;
    const double *in = buf + (plus ? 0 : n_per);
    f.base[(long long)l * f.sl + (long long)col * f.sx + (long long)y * f.sy] =
        in[(long long)kk * NY + y];
}

static int ring_pack(const TlbField *f, int ymode, double *sbuf, cudaStream_t s) {
    FaceLines tp = face_lines(1, 0), tm = face_lines(-1, 0);
    const int NY = f->Ly + 2 * f->Hy;
    dim3 grid((NY + 127) / 128, tp.n + tm.n);
    k_pack2<<<grid, 128, 0, s>>>(mkfld(f), tp, tm, ymode, sbuf, tp.n * NY);
    return launch_check("ring pack");
}

static int ring_unpack(const TlbField *f, const double *rbuf, cudaStream_t s) {
    FaceLines tp = face_lines(1, 0), tm = face_lines(-1, 0);
    const int NY = f->Ly + 2 * f->Hy;
    dim3 grid((NY + 127) / 128, tp.n + tm.n);
    k_unpack2<<<grid, 128, 0, s>>>(mkfld(f), tp, tm, rbuf, tp.n * NY);
    return launch_check("ring unpack");
}

static int ring_exchange(TlbRing *r, size_t n_per, const double *sbuf, double *rbuf,
                         cudaStream_t s) {
    auto &N = tlbring::nccl();
    // data travelling +x goes to the right neighbour and arrives from the left
    TLB_NCCL_CHECK(N.GroupStart());
    TLB_NCCL_CHECK(N.Send(sbuf, n_per, ncclFloat64, r->right, r->comm, s));
    TLB_NCCL_CHECK(N.Recv(rbuf, n_per, ncclFloat64, r->left, r->comm, s));
    TLB_NCCL_CHECK(N.Send(sbuf + n_per, n_per, ncclFloat64, r->left, r->comm, s));
    TLB_NCCL_CHECK(N.Recv(rbuf + n_per, n_per, ncclFloat64, r->right, r->comm, s));
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
    if (r->side) cudaStreamSynchronize(r->side);
    if (r->comm && N.ok) N.CommDestroy(r->comm);
    if (r->ev_pack) cudaEventDestroy(r->ev_pack);
    if (r->ev_done) cudaEventDestroy(r->ev_done);
    if (r->side) cudaStreamDestroy(r->side);
    delete r;
    return TLB_OK;
}

int tlb_ring_exchange(tlb_ring_t r, const TlbField *f, int ymode, double *sbuf, double *rbuf,
                      tlb_stream_t stream) {
    cudaStream_t s = (cudaStream_t)stream;
    int e;
    if ((e = ring_pack(f, ymode, sbuf, s))) return e;
    const size_t n_per = (size_t)tlb_face_payload_len(f);
    if ((e = ring_exchange(r, n_per, sbuf, rbuf, s))) return e;
    return ring_unpack(f, rbuf, s);
}

int tlb_ring_step(tlb_ring_t r, const TlbField *prv, const TlbField *nxt, const TlbParams *p,
                  int flags, TlbStatus *status, double *sbuf, double *rbuf,
                  void *ev_bulk0, void *ev_bulk1, tlb_stream_t stream) {
    int e;
    if ((e = check_stencil())) return e;
    if ((e = check_params(p))) return e;
    if (flags & TLB_F_WRAP_X)
        return fail(TLB_ERR_CONTRACT, "ring step: X halos come from the neighbours");
    cudaStream_t s = (cudaStream_t)stream;
    const int h = TLB_WALL_ROWS;
    const int ymode = (flags & TLB_F_CLAMP_Y) ? 1 : (flags & TLB_F_WRAP_Y) ? 2 : 0;
    // 1. faces out of prv (Y halos sourced as the reference's pack would see them)
    if ((e = ring_pack(prv, ymode, sbuf, s))) return e;
    TLB_CUDA_CHECK(cudaEventRecord(r->ev_pack, s));
    TLB_CUDA_CHECK(cudaStreamWaitEvent(r->side, r->ev_pack, 0));
    // 2. exchange on the side stream
    const size_t n_per = (size_t)tlb_face_payload_len(prv);
    if ((e = ring_exchange(r, n_per, sbuf, rbuf, r->side))) return e;
    // 3. bulk columns on the main stream, concurrent with the exchange
    if (ev_bulk0) TLB_CUDA_CHECK(cudaEventRecord((cudaEvent_t)ev_bulk0, s));
    if (prv->Lx > 2 * h) {
        TlbRegion bulk = {prv->Hx + h, prv->Hx + prv->Lx - h, prv->Hy, prv->Hy + prv->Ly};
        if ((e = tlb_fused(prv, nxt, bulk, p, flags, status, s))) return e;
    }
    if (ev_bulk1) TLB_CUDA_CHECK(cudaEventRecord((cudaEvent_t)ev_bulk1, s));
    // 4. halos in, then the 3+3 border columns (one launch) on the side stream
    if ((e = ring_unpack(prv, rbuf, r->side))) return e;
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
        const int wl = prv->Lx > 2 * h ? h : prv->Lx;
        Rect rs[2] = {mkrect(prv->Hx, prv->Hx + wl, prv->Hy, prv->Hy + prv->Ly),
                      mkrect(prv->Hx + prv->Lx - h, prv->Hx + prv->Lx, prv->Hy,
                             prv->Hy + prv->Ly)};
        set_frames(L, rs, prv->Lx > 2 * h ? 2 : 1);
        if ((e = launch_site<K_FUSED, false>(L, p->arith == TLB_ARITH_EXACT, p->order, r->side,
                                             "ring borders")))
            return e;
    }
    // 5. join
    TLB_CUDA_CHECK(cudaEventRecord(r->ev_done, r->side));
    TLB_CUDA_CHECK(cudaStreamWaitEvent(s, r->ev_done, 0));
    return TLB_OK;
}

}  // extern "C"
