/*
 * tlb.h -- C ABI of the B200-native D2Q37 thermal lattice-Boltzmann step
 * (libtlb.so, built from paper_1703_00185_b200/csrc/).
 *
 * The reference (`thermolb`, /root/reference/pkg/src/thermolb) has no FFI:
 * its hot path is plain Python functions.  Each entry point below replaces
 * one of them; the Python mirror (paper_1703_00185_b200/kernels.py,
 * runtime.py) keeps the reference signatures and calls these through ctypes.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Field memory is owned by the caller
 *    (torch tensors on the host side); the library never allocates fields.
 *  - A field is a strided (Q=37, NX, NY) view: element (l, x, y) lives at
 *    base[l*sl + x*sx + y*sy] (the reference's canonical view,
 *    geometry.py:95-100; SoA canonical strides are (NX*NY, NY, 1),
 *    geometry.py:72-73).  Coordinates are padded (halo-inclusive).
 *  - Regions are half-open [x0,x1) x [y0,y1) in padded coordinates and must
 *    lie inside the physical region (kernels.py:149-156) or the call returns
 *    TLB_ERR_CONTRACT.  An empty region is a no-op (kernels.py:221-222).
 *  - All compute calls are stream-ordered and asynchronous.  Per-site
 *    failures (non-positive density, T_bar <= 0, bad wall state) are written
 *    to a caller-owned device status block (TlbStatus) and surface when the
 *    host reads it; the host layer raises the errors.py exception.
 *  - Return value: 0 = ok, else a TLB_ERR_* code; message via
 *    tlb_last_error().
 */
#ifndef TLB_H
#define TLB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *tlb_stream_t; /* == cudaStream_t */

#define TLB_Q 37
#define TLB_WALL_ROWS 3 /* kernels.py:18 */

/* return codes */
#define TLB_OK 0
#define TLB_ERR_CONTRACT 1    /* ContractViolation (bad region/index)      */
#define TLB_ERR_CUDA 2        /* CUDA runtime error                        */
#define TLB_ERR_STENCIL 3     /* stencil not set / not the D2Q37 ordering  */
#define TLB_ERR_UNSUPPORTED 4 /* UnsupportedCaseError                      */
#define TLB_ERR_DOMAIN 5      /* DomainError detected on the host          */

/* device status bits (TlbStatus.flags), checked by the host */
#define TLB_ST_DEGENERATE 1u /* rho <= 0 (or NaN) in moments  kernels.py:62-66  */
#define TLB_ST_SHIFT 2u      /* T_bar <= 0 in apply_shift     kernels.py:134-135 */
#define TLB_ST_EQ_DOMAIN 4u  /* rho<=0 or T<=0, checked eq.   kernels.py:85-86   */
#define TLB_ST_PEER_TIMEOUT 8u /* peer step: a neighbour did not publish in time */
#define TLB_ST_PROTOCOL 16u    /* halo from a mis-sequenced step  runtime.py:151-154 */

/* field view */
typedef struct TlbField {
    double *base;           /* element (0, 0, 0)                            */
    int64_t sl, sx, sy;     /* strides (elements) of l, x, y                */
    int32_t Lx, Ly, Hx, Hy; /* physical extents and halo widths             */
} TlbField;

/* physics (kernels.py:21-38); D is fixed to 2 */
typedef struct TlbParams {
    double tau, gx, gy, dt;
    double Twall_top, Twall_bot;
    int32_t order; /* Hermite order 2, 3 or 4 (4 = D2Q37 default)          */
    int32_t arith; /* TLB_ARITH_EXACT (bitwise = reference) or _FAST       */
} TlbParams;

#define TLB_ARITH_EXACT 0
#define TLB_ARITH_FAST 1

typedef struct TlbRegion {
    int32_t x0, x1, y0, y1;
} TlbRegion;

/* caller-owned DEVICE memory, zero-initialised by the caller */
typedef struct TlbStatus {
    uint32_t flags;          /* OR of TLB_ST_* bits                          */
    int32_t site_x[3];       /* first (by atomic race) failing site per bit  */
    int32_t site_y[3];
    int32_t step;            /* step tag of the first failure (-1 unknown)   */
    uint32_t pad;
    unsigned long long negatives; /* count of f<0 written (count_negative) */
} TlbStatus;

/* step flags for tlb_fused / tlb_step */
#define TLB_F_WALL_BOT 1   /* bc rows [Hy, Hy+3) at Twall_bot before collide  */
#define TLB_F_WALL_TOP 2   /* bc rows [Hy+Ly-3, Hy+Ly) at Twall_top            */
#define TLB_F_CLAMP_BOT 4  /* read the bottom Y halo as the wall-row extension (runtime.py:296-305) */
#define TLB_F_WRAP_X 8     /* read X halo periodically (self ring, Np = 1)     */
#define TLB_F_WRAP_Y 16    /* read Y halo periodically (periodic_y)            */
#define TLB_F_COUNT_NEG 32 /* add count of written f<0 to status->negatives    */
#define TLB_F_CLAMP_TOP 64 /* read the top Y halo as the wall-row extension    */
#define TLB_F_CLAMP_Y (TLB_F_CLAMP_BOT | TLB_F_CLAMP_TOP)
#define TLB_F_POISON_HALOS 128 /* peer step, debug: NaN prv's halos once read (runtime.py:288-294) */

/* library */
int tlb_version(void);
const char *tlb_last_error(void);
int tlb_set_device(int device);
int tlb_device_count(void);

/* Upload the stencil constants to `device`.  c is (37,2) int64 in the
 * reference ordering (velocity_set.py:55-59), w (37,) the weights, cs2 the
 * squared sound speed -- all as built by velocity_set.build_velocity_set
 * (velocity_set.py:128-130).  ex = c/cs and q = ex^2+ey^2 are derived here
 * with the expressions of kernels.py:87-97.  Returns TLB_ERR_STENCIL if c is
 * not the D2Q37 ordering or w is not constant per speed shell. */
int tlb_set_stencil(int device, const int64_t *c, const double *w, double cs2);

/* Any stencil of Q <= 37 populations (e.g. D2Q9, velocity_set.py:117-124):
 * the reference D2Q37 ordering selects the specialised kernels, anything
 * else the generic per-population kernels (csrc/generic.cuh: the reference
 * arithmetic, bitwise; "fast" falls back to it).  Built for Q = 9 and 37. */
int tlb_set_stencil_q(int device, int q, const int64_t *c, const double *w,
                      double cs2);
/* test hook: run the D2Q37 stencil through the generic kernels (1) or the
 * specialised ones (0) */
int tlb_force_generic(int device, int on);

/* propagate (pull)      replaces kernels.propagate, kernels.py:168-177 */
int tlb_propagate(const TlbField *prv, const TlbField *nxt, TlbRegion r,
                  tlb_stream_t stream);

/* bc (wall rows)        replaces kernels.bc, kernels.py:180-203.
 * Columns [x0, x1); top/bottom select the walls. */
int tlb_bc(const TlbField *f, const TlbParams *p, int top, int bottom,
           int32_t x0, int32_t x1, TlbStatus *status, tlb_stream_t stream);

/* collide (in place allowed: in == out)   replaces kernels.collide,
 * kernels.py:139-146, on the region of a field (runtime.py:322-324) or on a
 * (Q, nx, ny) block described as a halo-free field. */
int tlb_collide(const TlbField *in, const TlbField *out, TlbRegion r,
                const TlbParams *p, int flags, TlbStatus *status,
                tlb_stream_t stream);

/* fused propagate(+bc)+collide   replaces kernels.propagate_collide_fused,
 * kernels.py:206-224, extended with bc on wall rows (RankWorker._tb_frame,
 * runtime.py:340-353) so one launch is a full staged step on its region. */
int tlb_fused(const TlbField *prv, const TlbField *nxt, TlbRegion r,
              const TlbParams *p, int flags, TlbStatus *status,
              tlb_stream_t stream);

/* One whole time step of a rank whose X ring neighbours are itself
 * (Np = 1) and whose Y direction has walls or is periodic: a single fused
 * launch over the physical region with implicit halos (WRAP_X + CLAMP_Y or
 * WRAP_Y).  Bitwise equal to RankWorker.step (runtime.py:355-400). */
int tlb_step_self(const TlbField *prv, const TlbField *nxt,
                  const TlbParams *p, int walls, int periodic_y,
                  int count_neg, TlbStatus *status, tlb_stream_t stream);

/* TWO whole time steps of such a rank in one launch (temporal blocking,
 * csrc/tb2.cu): prv -> nxt after steps `step` and `step`+1, the intermediate
 * state kept in shared memory.  Bitwise equal to two tlb_step_self calls;
 * status1/status2 receive the per-step failures and negative counts.
 * D2Q37 order 4, tiles of at least 8x8 (else TLB_ERR_UNSUPPORTED). */
int tlb_step2_self(const TlbField *prv, const TlbField *nxt,
                   const TlbParams *p, int walls, int periodic_y,
                   int count_neg, TlbStatus *status1, TlbStatus *status2,
                   int step, tlb_stream_t stream);

/* moments               replaces kernels.moments, kernels.py:41-71.
 * Outputs are (nx, ny) arrays with row stride ld (elements). */
int tlb_moments(const TlbField *f, TlbRegion r, double *rho, double *ux,
                double *uy, double *T, int64_t ld, int check,
                TlbStatus *status, tlb_stream_t stream);

/* equilibrium           replaces kernels.equilibrium, kernels.py:74-125,
 * on n sites; out is (37, n) with leading dimension ld. */
int tlb_equilibrium(const double *rho, const double *ux, const double *uy,
                    const double *T, int64_t n, int order, int arith,
                    double *out, int64_t ld, int check, TlbStatus *status,
                    tlb_stream_t stream);

/* apply_shift           replaces kernels.apply_shift, kernels.py:128-136 */
int tlb_apply_shift(const double *ux, const double *uy, const double *T,
                    int64_t n, const TlbParams *p, double *ub, double *vb,
                    double *Tb, TlbStatus *status, tlb_stream_t stream);

/* count_negative        replaces kernels.count_negative, kernels.py:227-229 */
int tlb_count_negative(const TlbField *f, TlbRegion r, TlbStatus *status,
                       tlb_stream_t stream);

/* _extend_wall_halos    replaces RankWorker._extend_wall_halos,
 * runtime.py:296-305 (all x, all 37 populations). */
int tlb_extend_walls(const TlbField *f, int upper, int lower,
                     tlb_stream_t stream);

/* Face-plan X payloads  replace RankWorker.pack_x / unpack_x,
 * runtime.py:199-224 (plans runtime.py:94-107): for d = 1..3, for l with
 * sign*c_l,x >= d in ascending l, one full-height column of NY values.
 * ymode selects how Y-halo rows are sourced when packing: 0 = memory as is
 * (the reference), 1 = wall extension (clamp) at both walls, 2 = periodic
 * wrap, 3 = clamp the bottom only, 4 = clamp the top only (2-D wall ranks). */
int64_t tlb_face_payload_len(const TlbField *f); /* 26 * NY */
int tlb_pack_x(const TlbField *f, int sign, int ymode, double *buf,
               tlb_stream_t stream);
int tlb_unpack_x(const TlbField *f, int sign, const double *buf,
                 tlb_stream_t stream);

/* Face-plan Y payloads (2-D tiling) replace RankWorker.pack_y / unpack_y,
 * runtime.py:226-246: for e = 1..3, for l with sign*c_l,y >= e in ascending
 * l, the row Hy+Ly-e (sign +1) or Hy+e-1 (sign -1) over the Lx physical
 * columns; unpack writes row Hy-e (+1, from below) or Hy+Ly-1+e (-1). */
int64_t tlb_face_payload_len_y(const TlbField *f); /* 26 * Lx */
int tlb_pack_y(const TlbField *f, int sign, double *buf, tlb_stream_t stream);
int tlb_unpack_y(const TlbField *f, int sign, const double *buf,
                 tlb_stream_t stream);

/* pbc_c / pbc_nc with the rank as its own neighbour (1-D ring of one rank;
 * periodic Y): runtime.py:248-284. */
int tlb_pbc_self_x(const TlbField *f, tlb_stream_t stream);
int tlb_pbc_self_y(const TlbField *f, tlb_stream_t stream);

/* Fill a field's X halo columns (face-plan populations, all NY rows) from
 * peer fields: left neighbour's right edge -> low-x halo, right neighbour's
 * left edge -> high-x halo.  Pointers may be peer-mapped (NVLink). */
int tlb_halo_from_peers(const TlbField *f, const TlbField *left,
                        const TlbField *right, tlb_stream_t stream);

/* ---- 1-D X ring across GPUs (one process per GPU) ----------------------
 * Replaces Fabric + pbc_c + the overlapped RankWorker.step for ranks on
 * different GPUs (runtime.py:116-160, 269-284, 378-396).  NCCL is loaded at
 * run time (libnccl.so.2 -- the copy PyTorch already loaded, if any). */
typedef struct TlbRing *tlb_ring_t;

int tlb_nccl_version(int *version);
/* 128-byte ncclUniqueId, created on rank 0 and broadcast by the caller */
int tlb_nccl_unique_id(char *out128);
/* left = rank-1, right = rank+1 (mod nranks), runtime.py:76-77 */
int tlb_ring_create(const char *uid128, int nranks, int rank, int device,
                    tlb_ring_t *out);
int tlb_ring_destroy(tlb_ring_t ring);
/* Failure detection (runtime.py:146-160 analog): the communicator's async
 * NCCL error (0 = ncclSuccess), and an abort that releases stalled NCCL
 * kernels so a rank that timed out can raise and exit. */
int tlb_ring_async_error(tlb_ring_t ring, int *nccl_result);
int tlb_ring_abort(tlb_ring_t ring);
/* 2-D tiling (decompose, runtime.py:54-91): neighbour ranks in the NCCL
 * communicator; -1 = none (wall side).  With up/down neighbours the step
 * exchanges Y faces first (physical columns), then X faces (full height, so
 * corner halos carry diagonal data, runtime.py:8-12).  ybuf holds the two
 * Y payloads (tlb_face_payload_len_y each) for sending and two for
 * receiving: 4 * (26 * Lx + 1) doubles (each payload ends with its step
 * tag). */
int tlb_ring_set_neighbors(tlb_ring_t ring, int left, int right, int up,
                           int down, double *ybuf);
/* pack both X faces of f (ymode as tlb_pack_x), exchange with the ring
 * neighbours, unpack into the X halo columns; sbuf/rbuf hold 2 payloads
 * of tlb_face_payload_len + 1 doubles each (+x face first; the last double
 * of each is the sender's step tag). */
int tlb_ring_exchange(tlb_ring_t ring, const TlbField *f, int ymode,
                      double *sbuf, double *rbuf, tlb_stream_t stream);
/* One overlapped time step: pack -> NCCL exchange (side stream) || bulk
 * fused kernel (stream) -> unpack + border columns (side stream) -> join.
 * flags as tlb_fused without TLB_F_WRAP_X.  ev_bulk0/1 (cudaEvent_t or NULL)
 * are recorded around the bulk kernel on `stream`.  step_tag travels with
 * every payload; a received tag other than ours sets TLB_ST_PROTOCOL
 * (Fabric.recv's step check, runtime.py:151-154). */
int tlb_ring_step(tlb_ring_t ring, const TlbField *prv, const TlbField *nxt,
                  const TlbParams *p, int flags, TlbStatus *status,
                  double *sbuf, double *rbuf, void *ev_bulk0, void *ev_bulk1,
                  int64_t step_tag, tlb_stream_t stream);

/* ---- X-halo exchange fused into the step over NVLink peer memory --------
 * (1-D ring or 2-D grid, one process per GPU; runtime.py:226-284 pbc_nc /
 * pbc_c + :355-400 step).
 * One kernel per step: the border threads store their outputs locally and
 * the face-plan lines (runtime.py:94-107) into the neighbours' nxt halo
 * columns through CUDA-IPC mapped pointers; the last border block to finish
 * publishes the step into the neighbours' mailboxes (st.release.sys); border
 * blocks of the next step wait for both neighbours (bounded; sticky
 * TLB_ST_PEER_TIMEOUT on expiry).  Replaces pack -> NCCL -> unpack of
 * tlb_ring_step. */
typedef struct TlbPeer *tlb_peer_t;
/* 64-byte cudaIpcMemHandle of the allocation holding ptr, and ptr's offset */
int tlb_ipc_handle(const void *ptr, char *out64, int64_t *offset);
/* Neighbours across processes: 8 directions d = left, right, down, up,
 * down-left, down-right, up-left, up-right (a 1-D X ring marks left and
 * right only); handles/offsets hold (A, B, mailbox) per direction (24 each),
 * A = the buffer that is prv at even peer steps; present[8] marks the
 * exchanged directions (others ignored). */
int tlb_peer_create2(int device, const char *handles, const int64_t *offsets,
                     const int *present, tlb_peer_t *out);
int tlb_peer_destroy(tlb_peer_t peer);
/* In-process neighbours (several ranks driven by one process, on one or
 * several GPUs): ptrs[3*d .. 3*d+2] = neighbour d's buffer A, buffer B and
 * mailbox (plain device pointers); peer access is enabled where needed. */
int tlb_peer_create_local(int device, void *const *ptrs, const int *present,
                          tlb_peer_t *out);
/* Bound of the border blocks' wait for a neighbour (default 5 s); the host
 * passes its fabric timeout (SimConfig.recv_timeout, sim.py:40). */
int tlb_peer_set_timeout(tlb_peer_t peer, double seconds);
/* One step.  nxt_index: 0 if nxt is buffer A, 1 if B.  mailbox: this rank's
 * zeroed device mailbox of >= 11 u64 ([0..7] value published by the
 * neighbour in direction d, [8] border-block counter, [9] sticky failure, [10]
 * the two-step ring kernel's work counter).
 * peer_step: 0, 1, 2, ... (border blocks wait for mailbox count >=
 * peer_step).  step_tag: the step number, published with the step and
 * checked against the neighbours' (TLB_ST_PROTOCOL on a mismatch, the
 * ProtocolError of Fabric.recv, runtime.py:151-154); check_prev: our
 * previous launch was step step_tag-1, so a neighbour still at our count
 * must carry that tag too.  flags may add TLB_F_POISON_HALOS. */
int tlb_peer_step(tlb_peer_t peer, const TlbField *prv, const TlbField *nxt,
                  int nxt_index, const TlbParams *p, int flags,
                  TlbStatus *status, unsigned long long *mailbox,
                  int64_t peer_step, int64_t step_tag, int check_prev,
                  tlb_stream_t stream);
/* Halo fill before the first step after a (re)load: the border sites push
 * their prv values into the neighbours' prv halos (exactly the lines the
 * step pushes) and publish as step step_tag (= first step - 1); counts as a
 * peer step.  prv_index: 0 if prv is buffer A, 1 if B. */
int tlb_peer_prime(tlb_peer_t peer, const TlbField *prv, int prv_index,
                   const TlbParams *p, TlbStatus *status,
                   unsigned long long *mailbox, int64_t peer_step,
                   int64_t step_tag, tlb_stream_t stream);

/* Two time steps per launch on a 1-D X ring (temporal blocking across
 * GPUs): the step-pair kernel of tlb_step2_self whose border runs read 6-column
 * X halos (prv->Hx >= 6) and store their own 6 border columns of the second
 * step into the neighbours' nxt halos (NVLink stores), with the mailbox
 * protocol of tlb_peer_step (one launch = one peer step; step_tag = the
 * first of the two steps; a neighbour's previous launch must have ended at
 * step_tag - 1).  Left and right neighbours only; Lx >= 12.  status1 /
 * status2: steps step_tag and step_tag + 1. */
int tlb_peer_step2(tlb_peer_t peer, const TlbField *prv, const TlbField *nxt,
                   int nxt_index, const TlbParams *p, int flags, TlbStatus *status1,
                   TlbStatus *status2, unsigned long long *mailbox, int64_t peer_step,
                   int64_t step_tag, int check_prev, tlb_stream_t stream);
/* Halo fill for tlb_peer_step2 (6 columns deep) before its first launch
 * after a (re)load or after single steps; counts as a peer step published
 * as step step_tag. */
int tlb_peer_prime2(tlb_peer_t peer, const TlbField *prv, int prv_index,
                    const TlbParams *p, TlbStatus *status, unsigned long long *mailbox,
                    int64_t peer_step, int64_t step_tag, tlb_stream_t stream);

/* Snapshot image (io.write_pgm, io.py:13-24): min-max normalised 8-bit
 * quantisation of a (nx, ny) field with row stride ld into img (nx*ny bytes,
 * PGM row order: top row = largest y).  minmax2 is 2 x u64 device scratch. */
int tlb_pgm_image(const double *v, int64_t nx, int64_t ny, int64_t ld,
                  unsigned long long *minmax2, unsigned char *img,
                  tlb_stream_t stream);

/* Tuning knobs (process-wide): TLB_TUNE_MINBLOCKS selects the
 * __launch_bounds__ minimum CTAs/SM of the fused kernel (1 = compiler's
 * choice, 4 = default, 5). */
#define TLB_TUNE_MINBLOCKS 1
#define TLB_TUNE_TB2_CFG 2   /* two-step kernel shape (rows x columns per iteration,
                                CTAs/SM): 0 = 128 x 2, 1; 1 = 64 x 2, 2 (default);
                                2 = 96 x 2, 1; 3-6 warp-specialised variants;
                                7 = 64 x 2, 2, one site on two threads (fast
                                arithmetic; exact runs shape 1) */
#define TLB_TUNE_TB2_RUN 3   /* two-step kernel: columns per work item (0 = chosen
                                per lattice to fill whole waves; default) */
#define TLB_TUNE_TB2_ORDER 4 /* two-step kernel work order: -1 auto (default: run-major
                                for fields >= 4 GB), 0 strip-major, 1 run-major
                                (all strips at one X range first) */
int tlb_set_tuning(int key, int value);
/* Current value of a tuning knob. */
int tlb_get_tuning(int key, int *value);

/* Diagnostics: measured FP64 FMA throughput of this GPU (flop/s, 2 per
 * DFMA), the denominator of the collide FP64 roofline. */
int tlb_bench_dfma(int64_t iters, double *flops_per_s, tlb_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* TLB_H */
