// tb2.cu -- two time steps per launch (temporal blocking): for a tile that
// is its own X neighbour (one rank: the BASELINE configs[1] step) and, with
// PEER, for a rank of the 1-D X ring of GPUs (configs[2]/[3]: 6-column X
// halos, border runs exchanging over NVLink -- see item_of_peer below).
//
// The single-step fused kernel moves the algorithmic minimum of ONE step
// (592 B/site) at the HBM roofline; the only way past it is to stop writing
// the intermediate state to HBM.  Here each CTA owns a strip of at most
// ROWS - 6 output rows (58 in the default 64 x 2 shape) and marches along X
// over a run of columns:
//
//   level 1 (step s):   a column of ROWS = HS + 6 sites (the strip plus 3
//                       rows of halo each side) is gathered from the level-0
//                       field in HBM (implicit periodic-X / wall-clamped or
//                       periodic-Y halos, exactly as the fused kernel),
//                       bc + collide in registers, and stored into a
//                       shared-memory ring;
//   level 2 (step s+1): the column 3 behind is gathered from the ring (the
//                       pull of propagate, kernels.py:168-177, served from
//                       shared memory), bc + collide, and streamed to HBM.
//
// Level-1 rows outside the lattice are materialised in the ring as the
// reference's halos of the intermediate state would be: wall ranks' halo rows
// are the extension of the first/last physical row (_extend_wall_halos,
// runtime.py:296-305: the thread computes that physical site), periodic Y
// wraps.  Per site update that is 296 B read + 296 B written per TWO steps
// (plus ~5 % strip/run overlap), against 592 B per step.
//
// The ring keeps population l of a level-1 column only as long as level 2
// needs it: column X is read by level-2 column X + c_x, so the ring of the
// populations with c_x = c is LANES + 3 + c columns deep (185 column slots
// for LANES = 2: 185 KB at 128 rows, one CTA of 8 warps per SM).  Columns
// are processed LANES at a time; the level-0 gather of the next columns is
// issued before the level-2 half so its HBM latency hides behind it.  Work
// items are runs of columns of one strip, handed out dynamically (an atomic
// counter); each run starts with a 3-column warm-up.
//
// Parity: the same per-site arithmetic as the fused kernel (d2q37.cuh), so
// two steps here are bitwise two fused steps (exact) -- tests compare with
// the C oracle.  Negatives (count_negative, kernels.py:227-229) are counted
// per step for the owned sites only; per-site failures are reported with
// their step.
#include <cuda_runtime.h>

#include "common.cuh"
#include "d2q37.cuh"
#include "tb2.cuh"

namespace tlb {
namespace tb2 {

// populations with c_x = c (c = -3..3), their ring depth and base slot
__host__ __device__ constexpr int GN(int c) {
    constexpr int t[7] = {3, 5, 7, 7, 7, 5, 3};
    return t[c + 3];
}
template <int LANES>
__host__ __device__ constexpr int GD(int c) { return LANES + 3 + c; }
template <int LANES>
__host__ __device__ constexpr int GBASE(int c) {
    int b = 0;
    for (int k = -3; k < c; ++k) b += GN(k) * GD<LANES>(k);
    return b;
}
__host__ __device__ constexpr int GIDX(int l) {
    int i = 0;
    for (int m = 0; m < l; ++m) i += CX(m) == CX(l);
    return i;
}
static_assert(GBASE<2>(4) == slots(2), "ring slots");

// slot (in units of ROWS doubles) of population l in ring column slot s
template <int LANES, int l>
__device__ __forceinline__ int slot_of(const int (&s)[7]) {
    return GBASE<LANES>(CX(l)) + s[CX(l) + 3] * GN(CX(l)) + GIDX(l);
}

// level-1 outputs go straight into the ring as they are produced
template <int ROWS, int LANES>
struct RingPut {
    double (&a)[Q];
    double *row;           // ring + this thread's row
    const int (&ws)[7];    // write slot per c_x group
    unsigned sgn;          // OR of the outputs' high words (sign_or)
    __device__ __forceinline__ double get(int l) const { return a[l]; }
    __device__ __forceinline__ void put(int l, double v) {
        switch (l) {
#define TLB_RP(L) case L: row[slot_of<LANES, L>(ws) * ROWS] = v; break;
            TLB_RP(0) TLB_RP(1) TLB_RP(2) TLB_RP(3) TLB_RP(4) TLB_RP(5) TLB_RP(6) TLB_RP(7)
            TLB_RP(8) TLB_RP(9) TLB_RP(10) TLB_RP(11) TLB_RP(12) TLB_RP(13) TLB_RP(14)
            TLB_RP(15) TLB_RP(16) TLB_RP(17) TLB_RP(18) TLB_RP(19) TLB_RP(20) TLB_RP(21)
            TLB_RP(22) TLB_RP(23) TLB_RP(24) TLB_RP(25) TLB_RP(26) TLB_RP(27) TLB_RP(28)
            TLB_RP(29) TLB_RP(30) TLB_RP(31) TLB_RP(32) TLB_RP(33) TLB_RP(34) TLB_RP(35)
            TLB_RP(36)
#undef TLB_RP
        }
        sgn = sign_or(sgn, v);
    }
    // exact count of outputs < 0, re-read from the ring only when a sign bit
    // was seen
    __device__ __forceinline__ unsigned negatives() const {
        return (int)sgn >= 0 ? 0u : count_slow();
    }
    __device__ __forceinline__ unsigned count_slow() const;
};

template <int ROWS, int LANES>
__device__ __forceinline__ unsigned RingPut<ROWS, LANES>::count_slow() const {
    unsigned n = 0;
#define TLB_RG(L) n += row[slot_of<LANES, L>(ws) * ROWS] < 0.0;
    TLB_RG(0) TLB_RG(1) TLB_RG(2) TLB_RG(3) TLB_RG(4) TLB_RG(5) TLB_RG(6) TLB_RG(7)
    TLB_RG(8) TLB_RG(9) TLB_RG(10) TLB_RG(11) TLB_RG(12) TLB_RG(13) TLB_RG(14)
    TLB_RG(15) TLB_RG(16) TLB_RG(17) TLB_RG(18) TLB_RG(19) TLB_RG(20) TLB_RG(21)
    TLB_RG(22) TLB_RG(23) TLB_RG(24) TLB_RG(25) TLB_RG(26) TLB_RG(27) TLB_RG(28)
    TLB_RG(29) TLB_RG(30) TLB_RG(31) TLB_RG(32) TLB_RG(33) TLB_RG(34) TLB_RG(35)
    TLB_RG(36)
#undef TLB_RG
    return n;
}

// level-2 outputs stream to HBM
struct GlobalPut {
    double (&a)[Q];
    char *dp;
    const long long *doffb;
    unsigned sgn;
    __device__ __forceinline__ double get(int l) const { return a[l]; }
    __device__ __forceinline__ void put(int l, double v) {
        *reinterpret_cast<double *>(dp + doffb[l]) = v;
        sgn = sign_or(sgn, v);
    }
    __device__ __forceinline__ unsigned negatives() const {
        return (int)sgn >= 0 ? 0u : count_slow();
    }
    // exact count, re-read from the thread's own stores (coherent loads)
    __device__ __forceinline__ unsigned count_slow() const {
        unsigned n = 0;
#pragma unroll 1
        for (int l = 0; l < Q; ++l)
            n += *reinterpret_cast<const volatile double *>(dp + doffb[l]) < 0.0;
        return n;
    }
};

template <int ROWS, int LANES, int l>
__device__ __forceinline__ void ring_get(double (&g)[Q], const double *row, const int (&rs)[7]) {
    g[l] = row[slot_of<LANES, l>(rs) * ROWS - CY(l)];
}
template <int ROWS, int LANES, int... Ls>
struct RingGet {
    __device__ __forceinline__ static void run(double (&g)[Q], const double *row,
                                               const int (&rs)[7]) {
        (ring_get<ROWS, LANES, Ls>(g, row, rs), ...);
    }
};

// level-0 gather for the level-1 site (x, y) (padded coordinates).  XWRAP:
// the tile is its own X neighbour (implicit periodic halo); else the X halo
// memory is read (the ring variant's 6 columns).  coh: coherent L2 loads for
// halos other GPUs stored while this grid may be running.
template <bool XWRAP>
__device__ __forceinline__ void gather0(double (&f)[Q], const TbLaunch &T, int x, int y,
                                        bool coh = false) {
    const Fld &S = T.src;
    const bool inner = (!XWRAP || (x >= S.Hx + 3 && x < S.Hx + S.Lx - 3)) && y >= S.Hy + 3 &&
                       y < S.Hy + S.Ly - 3;
    if (inner) {
        const char *sp = reinterpret_cast<const char *>(S.base + (long long)x * S.sx +
                                                        (long long)y * S.sy);
        // the ring variant takes the coherent path for every column: one load
        // sequence the compiler can hoist as a whole (a branch between an
        // .nc and a .cg copy cost the prefetch its overlap: long_scoreboard
        // 0.33 -> 1.63 per issue, profiles/r02_tb2.md)
        if (!XWRAP) {
#pragma unroll
            for (int l = 0; l < Q; ++l)
                f[l] = __ldcg(reinterpret_cast<const double *>(sp + T.soffb[l]));
        } else {
#pragma unroll
            for (int l = 0; l < Q; ++l)
                f[l] = __ldg(reinterpret_cast<const double *>(sp + T.soffb[l]));
        }
    } else if (!XWRAP || coh) {
        load_all<1>(f, S, x, y, true, true, T.flags);
    } else {
        load_all<0>(f, S, x, y, true, true, T.flags);
    }
}

template <bool EXACT>
__device__ __forceinline__ unsigned walls(double (&f)[Q], const TbLaunch &T, int y) {
    unsigned bits = 0;
    const bool bot = y >= T.bot_lo && y < T.bot_hi;
    const bool top = y >= T.top_lo && y < T.top_hi;
    if (bot || top) {
        // bottom wall then top wall, like bc() (kernels.py:190-203)
#pragma unroll 1
        for (int side = 0; side < 2; ++side) {
            if (!(side ? top : bot)) continue;
            const double Tw = side ? T.P.Ttop : T.P.Tbot;
            RegF rf{f};
            bits |= EXACT ? bc_exact<4>(rf, Tw) : bc_fast<4>(rf, Tw);
        }
    }
    return bits;
}

// Work item i -> (strip, first column, end column), padded coordinates.
// Wall strips (bc rows: slower per column) come first, in runs of half
// length, so the dynamic schedule ends on short uniform runs.
__device__ __forceinline__ void item_of(const TbLaunch &T, long long i, int &strip, int &xa,
                                        int &xb) {
    const int Lx = T.src.Lx;
    const long long nh = (long long)T.nheavy * T.hruns;
    if (i < nh) {
        const int h = (int)(i / T.hruns);
        strip = h == 0 ? 0 : T.ns - 1;
        const int r = (int)(i % T.hruns);
        xa = r * T.run_h;
        xb = xa + T.run_h < Lx ? xa + T.run_h : Lx;
    } else {
        i -= nh;
        int r;
        if (T.runmajor) {
            // concurrent CTAs share one X range of every strip: the address
            // span in flight stays ~run columns wide on huge tiles
            const int nl = T.ns - T.nheavy;
            strip = T.first_light + (int)(i % nl);
            r = (int)(i / nl);
        } else {
            strip = T.first_light + (int)(i / T.lruns);
            r = (int)(i % T.lruns);
        }
        xa = r * T.run_l;
        xb = xa + T.run_l < Lx ? xa + T.run_l : Lx;
    }
    xa += T.src.Hx;
    xb += T.src.Hx;
}

// Ring variant: the same runs; the border runs (first and last of every
// strip: they read the X halos and store into the neighbours) start the
// second wave -- late enough that the neighbours' previous launch (which
// ended about when ours did) has published, early enough that their
// slower coherent loads and remote stores do not form the launch's tail.
__device__ __forceinline__ void item_of_peer(const TbLaunch &T, long long i, int &strip,
                                             int &xa, int &xb, bool &edge) {
    const int Lx = T.src.Lx;
    const long long e0 = T.pe.first_edge;
    if (i >= e0 && i < e0 + T.pe.edges) i = T.pe.interior + (i - e0);   // a border run
    else if (i >= e0) i -= T.pe.edges;                                     // interior after
    const long long hi = (long long)T.nheavy * (T.hruns - 2);
    const long long li = (long long)(T.ns - T.nheavy) * (T.lruns - 2);
    int rl, r;
    edge = false;
    if (i < hi) {
        const int h = (int)(i / (T.hruns - 2));
        strip = h == 0 ? 0 : T.ns - 1;
        r = 1 + (int)(i % (T.hruns - 2));
        rl = T.run_h;
    } else if (i < hi + li) {
        i -= hi;
        if (T.runmajor) {
            const int nl = T.ns - T.nheavy;
            strip = T.first_light + (int)(i % nl);
            r = 1 + (int)(i / nl);
        } else {
            strip = T.first_light + (int)(i / (T.lruns - 2));
            r = 1 + (int)(i % (T.lruns - 2));
        }
        rl = T.run_l;
    } else {
        const long long j = i - hi - li;
        edge = true;
        strip = (int)(j / 2);
        const bool heavy = T.nheavy > 0 && (strip == 0 || strip == T.ns - 1);
        rl = heavy ? T.run_h : T.run_l;
        const int runs = heavy ? T.hruns : T.lruns;
        r = (j & 1) ? runs - 1 : 0;
    }
    xa = r * rl;
    xb = xa + rl < Lx ? xa + rl : Lx;
    xa += T.src.Hx;
    xb += T.src.Hx;
}

// thread 0: wait until both neighbours have published launch need-1;
// bit 0 = timeout / failed neighbour, bit 1 = step-tag mismatch
__device__ __forceinline__ int tb2_peer_wait(const TbPeer &E) {
    int fail = 0;
    const unsigned long long t0 = globaltimer();
    const unsigned long long need = (unsigned long long)E.need;
    for (int d = 0; d < 2 && !(fail & 1); ++d) {
        unsigned long long v;
        while (((v = ld_acquire_sys(E.mb + d)) & TLB_MB_CTR_MASK) < need) {
            if (ld_acquire_sys(E.mb + TLB_MB_STICKY) || globaltimer() - t0 > E.timeout_ns) {
                fail |= 1;
                break;
            }
            __nanosleep(256);
        }
        if (fail & 1) break;
        if (v & TLB_MB_POISON) {
            fail |= 1;
            break;
        }
        // a neighbour at our count ended at step tag - 1 (published tag), one
        // launch ahead at the end of this launch's span (tag + span)
        const unsigned long long ctr = v & TLB_MB_CTR_MASK;
        const unsigned long long tag = (v >> TLB_MB_TAG_SHIFT) & TLB_MB_TAG_MASK;
        if (need > 0) {
            if (ctr == need + 1) {
                if (tag != ((unsigned long long)(E.tag + E.span) & TLB_MB_TAG_MASK)) fail |= 2;
            } else if (ctr == need) {
                if (E.check_prev && tag != ((unsigned long long)E.tag & TLB_MB_TAG_MASK))
                    fail |= 2;
            } else {
                fail |= 2;
            }
        }
    }
    if (fail & 1) atomicExch(E.mb + TLB_MB_STICKY, 1ull);
    return fail;
}

// thread 0, after the block's border work: count it; the last border block
// publishes "launch done" (count need+1, tag = last step + 1) to both
// neighbours (fence / counter / fence, as in tlb_peer.cuh)
__device__ __forceinline__ void tb2_peer_done(const TbPeer &E, long long nblocks, long long tag_next) {
    __threadfence_system();
    if (atomicAdd(E.mb + TLB_MB_COUNTER, 1ull) != (unsigned long long)(nblocks - 1)) return;
    E.mb[TLB_MB_COUNTER] = 0;
    __threadfence_system();
    unsigned long long v = ((unsigned long long)E.need + 1) |
                           (((unsigned long long)tag_next & TLB_MB_TAG_MASK) << TLB_MB_TAG_SHIFT);
    if (ld_acquire_sys(E.mb + TLB_MB_STICKY)) v |= TLB_MB_POISON;
    // we are the left neighbour's right neighbour and vice versa
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(E.nbmb[0] + 1), "l"(v) : "memory");
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(E.nbmb[1] + 0), "l"(v) : "memory");
}

// level-2 outputs of a border column: also into the neighbour's halo, the
// populations its level-1 halo sites pull (depth d from our edge: left
// neighbour c_x <= 3 - d, right neighbour c_x >= d - 3)
struct PeerPut {
    double (&a)[Q];
    char *dp;
    const long long *doffb;
    char *lp, *rp;         // neighbours' site addresses (or null)
    int tl, tr;            // thresholds 3 - d (left), d - 3 (right)
    unsigned sgn;
    __device__ __forceinline__ double get(int l) const { return a[l]; }
    __device__ __forceinline__ void put(int l, double v) {
        *reinterpret_cast<double *>(dp + doffb[l]) = v;
        if (lp && CX(l) <= tl) *reinterpret_cast<double *>(lp + doffb[l]) = v;
        if (rp && CX(l) >= tr) *reinterpret_cast<double *>(rp + doffb[l]) = v;
        sgn = sign_or(sgn, v);
    }
    __device__ __forceinline__ unsigned negatives() const {
        if ((int)sgn >= 0) return 0u;
        unsigned n = 0;
#pragma unroll 1
        for (int l = 0; l < Q; ++l)
            n += *reinterpret_cast<const volatile double *>(dp + doffb[l]) < 0.0;
        return n;
    }
};

template <bool EXACT, int ROWS, int LANES, int MINB, bool PEER = false>
__global__ void __launch_bounds__(ROWS * LANES, MINB) k_tb2(const __grid_constant__ TbLaunch T) {
    extern __shared__ double ring[];
    __shared__ long long s_item;
    const int lane = threadIdx.x / ROWS, r = threadIdx.x % ROWS;
    const Fld &S = T.src;
    const int Lx = S.Lx, Ly = S.Ly, Hx = S.Hx, Hy = S.Hy;
    double *row = ring + r;
    unsigned neg1 = 0, neg2 = 0;
    __shared__ int s_fail;
    int fail = -1;           // ring variant: result of this block's one wait
    for (;;) {
        // dynamic schedule: the next work item (one strip run) for the CTA
        if (threadIdx.x == 0) s_item = (long long)atomicAdd(T.ctr, 1u);
        __syncthreads();
        const long long item = s_item;
        if (item >= T.items) break;
        int strip, xa, xb;
        bool edge = false;
        if constexpr (PEER) item_of_peer(T, item, strip, xa, xb, edge);
        else item_of(T, item, strip, xa, xb);
        if (PEER && edge && fail < 0) {
            // first border run of this block: both neighbours' previous
            // launch must be done (halos written, ours read)
            if (threadIdx.x == 0) s_fail = tb2_peer_wait(T.pe);
            __syncthreads();
            fail = s_fail;
            if (threadIdx.x == 0 && fail) {
                if (fail & 1) report(T.st1, TLB_ST_PEER_TIMEOUT, xa, Hy, T.step);
                if (fail & 2) report(T.st1, TLB_ST_PROTOCOL, xa, Hy, T.step);
            }
        }
        if (PEER && edge && (fail & 1)) {
            // a neighbour is gone: no compute, but count the run so the
            // (poisoned) publication still happens
            if (threadIdx.x == 0) tb2_peer_done(T.pe, T.pe.edges, T.step + 2);
            __syncthreads();     // every thread has read s_item before it is reused
            continue;
        }
        const int ys = Hy + (int)((long long)Ly * strip / T.ns);
        const int hs = Hy + (int)((long long)Ly * (strip + 1) / T.ns) - ys;
        // this thread's level-1 row and the physical site it stands for
        const int y1 = ys - 3 + r;
        const bool row1 = r < hs + 6;
        int y1s = y1;
        if (T.flags & TLB_F_WRAP_Y) {
            if (y1s < Hy) y1s += Ly;
            else if (y1s >= Hy + Ly) y1s -= Ly;
        } else {
            y1s = y1s < Hy ? Hy : (y1s >= Hy + Ly ? Hy + Ly - 1 : y1s);
        }
        const bool row2 = r >= 3 && r < hs + 3;   // level-2 row y1 is an output row
        const int K = (xb - xa + 6 + LANES - 1) / LANES;
        auto wrapx = [&](int x) {
            return PEER ? x : x < Hx ? x + Lx : (x >= Hx + Lx ? x - Lx : x);
        };
        double f[Q];
        // only gathers within 3 columns of a tile edge read the halos the
        // neighbours store: those (and only those) take the coherent path
        auto halo_col = [&](int x) { return PEER && edge && (x < Hx + 3 || x >= Hx + Lx - 3); };
        if (row1) gather0<!PEER>(f, T, wrapx(xa - 3 + lane), y1s, halo_col(xa - 3 + lane));
        // ring slots of level-1 column j (written) and of the columns level 2
        // reads (j - 3 - c), per c_x group; advanced by LANES per iteration
        int ws[7], rs[7];
#pragma unroll
        for (int c = -3; c <= 3; ++c) {
            ws[c + 3] = lane % GD<LANES>(c);
            rs[c + 3] = (lane + 2 * GD<LANES>(c) - 3 - c) % GD<LANES>(c);
        }
        for (int k = 0; k < K; ++k) {
            const int j = LANES * k + lane;      // ring column of this level-1 column
            const int X1 = xa - 3 + j;           // level-1 column (unwrapped)
            if (row1 && X1 < xb + 3) {
                const int xs = wrapx(X1);
                unsigned bits = walls<EXACT>(f, T, y1s);
                RingPut<ROWS, LANES> rp{f, row, ws, 0u};
                bits |= EXACT ? collide_exact<4>(rp, T.P) : collide_fast<4>(rp, T.P);
                if (bits) report(T.st1, bits, xs, y1s, T.step);
                if (row2 && X1 >= xa && X1 < xb) neg1 += rp.negatives();
            }
            // the next level-1 column's HBM gather, in flight during level 2
            if (row1 && k + 1 < K && X1 + LANES < xb + 3)
                gather0<!PEER>(f, T, wrapx(X1 + LANES), y1s, halo_col(X1 + LANES));
            __syncthreads();
            const int X2 = X1 - 3;
            if (row2 && X2 >= xa && X2 < xb) {
                double g[Q];
                RingGet<ROWS, LANES, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17,
                        18, 19, 20, 21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31, 32, 33, 34, 35,
                        36>::run(g, row, rs);
                unsigned bits = walls<EXACT>(g, T, y1);
                char *dp = reinterpret_cast<char *>(T.dst.base + (long long)X2 * T.dst.sx +
                                                    (long long)y1 * T.dst.sy);
                const int xp = X2 - Hx;
                const int dl = PEER && edge && xp < 6 ? xp + 1 : 0;
                const int dr = PEER && edge && xp >= Lx - 6 ? Lx - xp : 0;
                if (dl || dr) {
                    const long long off = (long long)y1 * T.dst.sy;
                    char *lp = dl ? reinterpret_cast<char *>(
                                        T.pe.nb[0] + (long long)(X2 + Lx) * T.dst.sx + off)
                                  : nullptr;
                    char *rp = dr ? reinterpret_cast<char *>(
                                        T.pe.nb[1] + (long long)(X2 - Lx) * T.dst.sx + off)
                                  : nullptr;
                    PeerPut pp{g, dp, T.doffb, lp, rp, 3 - dl, dr - 3, 0u};
                    bits |= EXACT ? collide_exact<4>(pp, T.P) : collide_fast<4>(pp, T.P);
                    neg2 += pp.negatives();
                } else {
                    GlobalPut gp{g, dp, T.doffb, 0u};
                    bits |= EXACT ? collide_exact<4>(gp, T.P) : collide_fast<4>(gp, T.P);
                    neg2 += gp.negatives();
                }
                if (bits) report(T.st2, bits, X2, y1, T.step + 1);
            }
#pragma unroll
            for (int c = -3; c <= 3; ++c) {
                ws[c + 3] += LANES;
                if (ws[c + 3] >= GD<LANES>(c)) ws[c + 3] -= GD<LANES>(c);
                rs[c + 3] += LANES;
                if (rs[c + 3] >= GD<LANES>(c)) rs[c + 3] -= GD<LANES>(c);
            }
            __syncthreads();
        }
        // a border run's halo reads and remote stores are done (the barrier
        // above): count it; the last one publishes
        if (PEER && edge && threadIdx.x == 0) tb2_peer_done(T.pe, T.pe.edges, T.step + 2);
    }
    if (T.flags & TLB_F_COUNT_NEG) {
        count_neg_n(T.st1, neg1);
        count_neg_n(T.st2, neg2);
    }
}

// Halo fill of the ring variant before its first launch after a (re)load:
// every rank pushes the populations of its 6 border columns of level 0 that
// the neighbours' level-1 halo sites pull into their level-0 halos (T.pe.nb
// = the neighbours' buffer twin of T.src), then publishes as a launch.
__global__ void k_tb2_prime(const __grid_constant__ TbLaunch T) {
    __shared__ int s_fail;
    if (threadIdx.x == 0) s_fail = tb2_peer_wait(T.pe);
    __syncthreads();
    const Fld &S = T.src;
    const long long n = 12LL * S.Ly;   // (side, depth) x rows
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (!(s_fail & 1) && i < n) {
        const int side = (int)(i / (6LL * S.Ly)), d = 1 + (int)((i / S.Ly) % 6);
        const int y = S.Hy + (int)(i % S.Ly);
        const int x = side ? S.Hx + S.Lx - d : S.Hx + d - 1;
        const long long so = (long long)x * S.sx + (long long)y * S.sy;
        const long long ro = (long long)(side ? x - S.Lx : x + S.Lx) * S.sx + (long long)y * S.sy;
        double *dst = T.pe.nb[side];
#pragma unroll
        for (int l = 0; l < Q; ++l) {
            const bool need = side ? CX(l) >= d - 3 : CX(l) <= 3 - d;
            if (need) dst[ro + (long long)l * S.sl] = S.base[so + (long long)l * S.sl];
        }
    }
    if (threadIdx.x == 0 && s_fail) {
        if (s_fail & 1) report(T.st1, TLB_ST_PEER_TIMEOUT, S.Hx, S.Hy, T.step);
        if (s_fail & 2) report(T.st1, TLB_ST_PROTOCOL, S.Hx, S.Hy, T.step);
    }
    __syncthreads();
    if (threadIdx.x == 0) tb2_peer_done(T.pe, gridDim.x, T.step + 1);
}

template <bool EXACT, int ROWS, int LANES, int MINB, bool PEER = false>
static cudaError_t launch_cfg(const TbLaunch &T, int sms, cudaStream_t s) {
    const size_t smem = (size_t)slots(LANES) * ROWS * sizeof(double);
    // the shared-memory opt-in is per device: one process may drive several
    static bool attr[64] = {};
    int dev = 0;
    cudaError_t e0 = cudaGetDevice(&dev);
    if (e0 != cudaSuccess) return e0;
    auto *fn = k_tb2<EXACT, ROWS, LANES, MINB, PEER>;
    if (dev < 0 || dev >= 64 || !attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < 64) attr[dev] = true;
    }
    long long grid = (long long)sms * MINB;
    if (grid > T.items) grid = T.items;
    fn<<<(unsigned)grid, ROWS * LANES, smem, s>>>(T);
    return cudaGetLastError();
}

// ------------------------------------------ split variant (fast, cfg 7) --
// The 64 x 2 kernel holds a whole site (37 populations in flight for the
// next level-0 column plus 37 for level 2) in 252 registers, so only 8 warps
// fit an SM and the FP64 chains stall on latency (profiles/r02_tb2.md).
// Here a site runs on two threads, one in each warp of a pair (warps 2p and
// 2p+1 hold the same 32 sites): half h owns the populations IN_HALF(h, l)
// (d2q37.cuh: 17 / 20 of them, about the same FP64 work), gathers, relaxes
// and stores only those, and the pair exchanges its partial moments through
// shared memory at a named barrier (ids 1-4).  At <= 128 registers two CTAs
// of 8 warps fit an SM: 16 warps, the same ring and strip geometry.
//
// Every thread of a pair must reach each exchange, so the per-row conditions
// only predicate stores and reports: threads on rows without work compute
// on whatever they hold (ring reads stay inside the 3-double pads).
constexpr int XSLOTS = 6;   // exchange slots: 4 moments, bottom and top wall rho

struct PairX {
    double *mine, *theirs;  // this thread's column of its half's / the partner's slots
    int pair;               // named barrier 1 + pair (immediate ids: ptxas then
                            // reserves 5 barriers per CTA, not all 16)
    template <int N>
    __device__ __forceinline__ void sum(double (&v)[N], int slot) {
#pragma unroll
        for (int k = 0; k < N; ++k) mine[(slot + k) * 32] = v[k];
        switch (pair) {
        case 0: asm volatile("bar.sync 1, 64;" ::: "memory"); break;
        case 1: asm volatile("bar.sync 2, 64;" ::: "memory"); break;
        case 2: asm volatile("bar.sync 3, 64;" ::: "memory"); break;
        default: asm volatile("bar.sync 4, 64;" ::: "memory"); break;
        }
#pragma unroll
        for (int k = 0; k < N; ++k) v[k] += theirs[(slot + k) * 32];
    }
};

// RingPut / GlobalPut for one half: the slow negatives recount covers only
// the half's own populations
template <int ROWS, int LANES, int H>
struct RingPutH : RingPut<ROWS, LANES> {
    __device__ __forceinline__ unsigned negatives() const {
        if ((int)this->sgn >= 0) return 0u;
        unsigned n = 0;
#define TLB_RG(L) if (IN_HALF(H, L)) n += this->row[slot_of<LANES, L>(this->ws) * ROWS] < 0.0;
        TLB_RG(0) TLB_RG(1) TLB_RG(2) TLB_RG(3) TLB_RG(4) TLB_RG(5) TLB_RG(6) TLB_RG(7)
        TLB_RG(8) TLB_RG(9) TLB_RG(10) TLB_RG(11) TLB_RG(12) TLB_RG(13) TLB_RG(14)
        TLB_RG(15) TLB_RG(16) TLB_RG(17) TLB_RG(18) TLB_RG(19) TLB_RG(20) TLB_RG(21)
        TLB_RG(22) TLB_RG(23) TLB_RG(24) TLB_RG(25) TLB_RG(26) TLB_RG(27) TLB_RG(28)
        TLB_RG(29) TLB_RG(30) TLB_RG(31) TLB_RG(32) TLB_RG(33) TLB_RG(34) TLB_RG(35)
        TLB_RG(36)
#undef TLB_RG
        return n;
    }
};

template <int H>
struct GlobalPutH {
    double (&a)[Q];
    char *dp;
    const long long *doffb;
    unsigned sgn;
    bool on;                // this thread's row is an output row
    __device__ __forceinline__ double get(int l) const { return a[l]; }
    __device__ __forceinline__ void put(int l, double v) {
        // a predicated store, not a branch per population
        asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p st.global.f64 [%0], %1; }" ::"l"(
                         dp + doffb[l]), "d"(v), "r"((unsigned)on) : "memory");
        sgn = sign_or(sgn, v);
    }
    __device__ __forceinline__ unsigned negatives() const {
        if ((int)sgn >= 0) return 0u;
        unsigned n = 0;
#pragma unroll 1
        for (int l = 0; l < Q; ++l)
            if (IN_HALF(H, l)) n += *reinterpret_cast<const volatile double *>(dp + doffb[l]) < 0.0;
        return n;
    }
};

template <int H, int l>
__device__ __forceinline__ void load_h(double (&f)[Q], const Fld &s, int x, int y, int flags) {
    if constexpr (IN_HALF(H, l)) load_one<l, false>(f, s, x, y, true, true, flags);
}
template <int H, int... Ls>
struct LoadHalf {
    __device__ __forceinline__ static void run(double (&f)[Q], const Fld &s, int x, int y,
                                               int flags) {
        (load_h<H, Ls>(f, s, x, y, flags), ...);
    }
};

template <int H>
__device__ __forceinline__ void gather0_half(double (&f)[Q], const TbLaunch &T, int x, int y) {
    const Fld &S = T.src;
    const bool inner = x >= S.Hx + 3 && x < S.Hx + S.Lx - 3 && y >= S.Hy + 3 &&
                       y < S.Hy + S.Ly - 3;
    if (inner) {
        const char *sp = reinterpret_cast<const char *>(S.base + (long long)x * S.sx +
                                                        (long long)y * S.sy);
#pragma unroll
        for (int l = 0; l < Q; ++l)
            if (IN_HALF(H, l)) f[l] = __ldg(reinterpret_cast<const double *>(sp + T.soffb[l]));
    } else {
        LoadHalf<H, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 21,
                 22, 23, 24, 25, 26, 27, 28, 29, 30, 31, 32, 33, 34, 35, 36>::run(f, S, x, y,
                                                                                  T.flags);
    }
}

template <int ROWS, int LANES, int l>
__device__ __forceinline__ void ring_get_h(double (&g)[Q], const double *row, const int (&rs)[7]) {
    g[l] = row[slot_of<LANES, l>(rs) * ROWS - CY(l)];
}
template <int H, int ROWS, int LANES, int... Ls>
struct RingGetHalf {
    __device__ __forceinline__ static void run(double (&g)[Q], const double *row,
                                               const int (&rs)[7]) {
        ((IN_HALF(H, Ls) ? ring_get_h<ROWS, LANES, Ls>(g, row, rs) : void()), ...);
    }
};

// bc on the wall rows of a wall strip: every thread exchanges (both sides,
// bottom then top like bc(), kernels.py:190-203), the rows in range apply
template <int H>
__device__ __forceinline__ unsigned walls_half(double (&f)[Q], const TbLaunch &T, int y,
                                               PairX &x) {
    unsigned bits = 0;
    const bool bot = y >= T.bot_lo && y < T.bot_hi;
    const bool top = y >= T.top_lo && y < T.top_hi;
    RegF rf{f};
    bits |= bc_fast_half<H, 4>(rf, T.P.Tbot, x, 4, bot);
    bits |= bc_fast_half<H, 4>(rf, T.P.Ttop, x, 5, top);
    return bits;
}

template <int H, int ROWS, int LANES, bool PF>
__device__ __forceinline__ void tb2s_body(const TbLaunch &T, double *ring, PairX &px, int lane,
                                          int r, long long &s_item, unsigned &neg1,
                                          unsigned &neg2) {
    const Fld &S = T.src;
    const int Lx = S.Lx, Ly = S.Ly, Hx = S.Hx, Hy = S.Hy;
    double *row = ring + r;
    for (;;) {
        if (threadIdx.x == 0) s_item = (long long)atomicAdd(T.ctr, 1u);
        __syncthreads();
        const long long item = s_item;
        if (item >= T.items) break;
        int strip, xa, xb;
        item_of(T, item, strip, xa, xb);
        const int ys = Hy + (int)((long long)Ly * strip / T.ns);
        const int hs = Hy + (int)((long long)Ly * (strip + 1) / T.ns) - ys;
        const int y1 = ys - 3 + r;
        const bool row1 = r < hs + 6;
        int y1s = y1;
        if (T.flags & TLB_F_WRAP_Y) {
            if (y1s < Hy) y1s += Ly;
            else if (y1s >= Hy + Ly) y1s -= Ly;
        } else {
            y1s = y1s < Hy ? Hy : (y1s >= Hy + Ly ? Hy + Ly - 1 : y1s);
        }
        const bool row2 = r >= 3 && r < hs + 3;
        // the strip's level-1 rows (clamped like y1s) meet a wall range:
        // uniform over the CTA, so the wall exchanges are too
        int lo = ys - 3, hi = ys + hs + 3;
        if (!(T.flags & TLB_F_WRAP_Y)) {
            lo = lo < Hy ? Hy : lo;
            hi = hi > Hy + Ly ? Hy + Ly : hi;
        }
        const bool wall = (lo < T.bot_hi && hi > T.bot_lo) || (lo < T.top_hi && hi > T.top_lo);
        const int K = (xb - xa + 6 + LANES - 1) / LANES;
        auto wrapx = [&](int x) { return x < Hx ? x + Lx : (x >= Hx + Lx ? x - Lx : x); };
        double f[Q];
        if (PF && row1) gather0_half<H>(f, T, wrapx(xa - 3 + lane), y1s);
        int ws[7], rs[7];
#pragma unroll
        for (int c = -3; c <= 3; ++c) {
            ws[c + 3] = lane % GD<LANES>(c);
            rs[c + 3] = (lane + 2 * GD<LANES>(c) - 3 - c) % GD<LANES>(c);
        }
        for (int k = 0; k < K; ++k) {
            const int j = LANES * k + lane;
            const int X1 = xa - 3 + j;
            if (X1 < xb + 3) {   // uniform over a warp (one column)
                if (!PF && row1) gather0_half<H>(f, T, wrapx(X1), y1s);
                unsigned bits = wall ? walls_half<H>(f, T, y1s, px) : 0u;
                RingPutH<ROWS, LANES, H> rp{{f, row, ws, 0u}};
                bits |= collide_fast_half<H, 4>(rp, T.P, px);
                if (H == 0 && row1 && bits) report(T.st1, bits, wrapx(X1), y1s, T.step);
                if (row2 && X1 >= xa && X1 < xb) neg1 += rp.negatives();
            }
            if (PF && row1 && k + 1 < K && X1 + LANES < xb + 3)
                gather0_half<H>(f, T, wrapx(X1 + LANES), y1s);
            __syncthreads();
            const int X2 = X1 - 3;
            if (X2 >= xa && X2 < xb) {   // uniform over a warp
                double g[Q];
                RingGetHalf<H, ROWS, LANES, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15,
                            16, 17, 18, 19, 20, 21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31, 32,
                            33, 34, 35, 36>::run(g, row, rs);
                unsigned bits = wall ? walls_half<H>(g, T, y1, px) : 0u;
                char *dp = reinterpret_cast<char *>(T.dst.base + (long long)X2 * T.dst.sx +
                                                    (long long)y1 * T.dst.sy);
                GlobalPutH<H> gp{g, dp, T.doffb, 0u, row2};
                bits |= collide_fast_half<H, 4>(gp, T.P, px);
                if (row2) {
                    neg2 += gp.negatives();
                    if (H == 0 && bits) report(T.st2, bits, X2, y1, T.step + 1);
                }
            }
#pragma unroll
            for (int c = -3; c <= 3; ++c) {
                ws[c + 3] += LANES;
                if (ws[c + 3] >= GD<LANES>(c)) ws[c + 3] -= GD<LANES>(c);
                rs[c + 3] += LANES;
                if (rs[c + 3] >= GD<LANES>(c)) rs[c + 3] -= GD<LANES>(c);
            }
            __syncthreads();
        }
    }
}

// shared memory: [3 pad][ring][3 pad][exchange: one XSLOTS x 32 block per warp
// (ROWS * LANES / 32 pairs x 2 halves)]
template <int ROWS, int LANES>
constexpr size_t split_smem() {
    return ((size_t)slots(LANES) * ROWS + 6 + (size_t)(2 * ROWS * LANES / 32) * XSLOTS * 32) *
           sizeof(double);
}

// PF: the next level-0 column is gathered into registers during level 2
template <int ROWS, int LANES, int MINB, bool PF>
__global__ void __launch_bounds__(2 * ROWS * LANES, MINB) k_tb2s(const __grid_constant__ TbLaunch T) {
    static_assert(ROWS % 32 == 0, "a warp covers 32 rows of one column");
    extern __shared__ double smem[];
    double *ring = smem + 3;
    double *xch = smem + slots(LANES) * ROWS + 6;
    const int warp = threadIdx.x / 32, h = warp & 1, p = warp >> 1;
    const int site = p * 32 + (threadIdx.x & 31);
    const int lane = site / ROWS, r = site % ROWS;
    double *col = xch + (size_t)p * 2 * XSLOTS * 32 + (threadIdx.x & 31);
    PairX px{col + h * XSLOTS * 32, col + (1 - h) * XSLOTS * 32, p};
    __shared__ long long s_item;
    unsigned neg1 = 0, neg2 = 0;
    if (h == 0) tb2s_body<0, ROWS, LANES, PF>(T, ring, px, lane, r, s_item, neg1, neg2);
    else tb2s_body<1, ROWS, LANES, PF>(T, ring, px, lane, r, s_item, neg1, neg2);
    if (T.flags & TLB_F_COUNT_NEG) {
        count_neg_n(T.st1, neg1);
        count_neg_n(T.st2, neg2);
    }
}

template <int ROWS, int LANES, int MINB, bool PF>
static cudaError_t launch_split(const TbLaunch &T, int sms, cudaStream_t s) {
    const size_t smem = split_smem<ROWS, LANES>();
    static bool attr[64] = {};
    int dev = 0;
    cudaError_t e0 = cudaGetDevice(&dev);
    if (e0 != cudaSuccess) return e0;
    auto *fn = k_tb2s<ROWS, LANES, MINB, PF>;
    if (dev < 0 || dev >= 64 || !attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < 64) attr[dev] = true;
    }
    long long grid = (long long)sms * MINB;
    if (grid > T.items) grid = T.items;
    fn<<<(unsigned)grid, 2 * ROWS * LANES, smem, s>>>(T);
    return cudaGetLastError();
}

// ------------------------------------------------ warp-specialised variant --
// Producer warps (level 1: HBM gather, bc + collide, ring) and consumer warps
// (level 2: ring gather, bc + collide, HBM) run concurrently.  They meet only
// at shared-memory mbarriers: full[column] (all ROWS producer threads of a
// level-1 column arrived) and empty[column] (all consumer threads of a
// level-2 column arrived), so no warp waits at a CTA-wide barrier inside a
// run.  The ring slack is E - 3 columns: the producer of level-1 column j
// may overwrite its slots once level-2 column j - E - 3 is done.
__device__ __forceinline__ void mb_init(unsigned long long *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_arrive(unsigned long long *b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long *b, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(b);
    unsigned done = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;"
                     " selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(a), "r"(parity) : "memory");
    } while (!done);
}

constexpr int NBAR = 32;   // full / empty barriers (column index mod NBAR)

template <bool EXACT, int ROWS, int PL, int CL, int E, int MINB>
__global__ void __launch_bounds__(ROWS * (PL + CL), MINB) k_tb2ws(const __grid_constant__ TbLaunch T) {
    constexpr int LANES = E - 3;        // ring depth of group c: E + c = GD<LANES>(c)
    constexpr int WPC = ROWS / 32;      // warps per column
    extern __shared__ double ring[];
    __shared__ unsigned long long full[NBAR], empty[NBAR];
    __shared__ long long s_item;
    const int warp = threadIdx.x / 32;
    const bool producer = warp < PL * WPC;
    const int lane = producer ? warp / WPC : (warp - PL * WPC) / WPC;
    const int r = (warp % WPC) * 32 + (threadIdx.x & 31);
    const Fld &S = T.src;
    const int Lx = S.Lx, Ly = S.Ly, Hx = S.Hx, Hy = S.Hy;
    double *row = ring + r;
    unsigned neg1 = 0, neg2 = 0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NBAR; ++i) {
            mb_init(&full[i], ROWS);               // every thread of the producing column
            mb_init(&empty[i], ROWS);              // every thread of the consuming column
        }
    }
    long long gj = 0, gm = 0;   // level-1 / level-2 columns of earlier runs (barrier phases)
    for (;;) {
        if (threadIdx.x == 0) s_item = (long long)atomicAdd(T.ctr, 1u);
        __syncthreads();        // also: the previous run has drained
        const long long item = s_item;
        __syncthreads();
        if (item >= T.items) break;
        int strip, xa, xb;
        item_of(T, item, strip, xa, xb);
        const int ys = Hy + (int)((long long)Ly * strip / T.ns);
        const int hs = Hy + (int)((long long)Ly * (strip + 1) / T.ns) - ys;
        const int y1 = ys - 3 + r;
        const int w = xb - xa, NJ = w + 6;
        auto wrapx = [&](int x) { return x < Hx ? x + Lx : (x >= Hx + Lx ? x - Lx : x); };
        if (producer) {
            const bool row1 = r < hs + 6;
            int y1s = y1;
            if (T.flags & TLB_F_WRAP_Y) {
                if (y1s < Hy) y1s += Ly;
                else if (y1s >= Hy + Ly) y1s -= Ly;
            } else {
                y1s = y1s < Hy ? Hy : (y1s >= Hy + Ly ? Hy + Ly - 1 : y1s);
            }
            const bool own_row = r >= 3 && r < hs + 3;
            for (int j = lane; j < NJ; j += PL) {
                const int X1 = xa - 3 + j;
                double f[Q];
                if (row1) gather0<true>(f, T, wrapx(X1), y1s);
                if (j >= E + 3) {
                    const long long m = gm + (j - E - 3);
                    mb_wait(&empty[m % NBAR], (unsigned)((m / NBAR) & 1));
                }
                if (row1) {
                    int wsl[7];
#pragma unroll
                    for (int c = -3; c <= 3; ++c) wsl[c + 3] = j % GD<LANES>(c);
                    unsigned bits = walls<EXACT>(f, T, y1s);
                    RingPut<ROWS, LANES> rp{f, row, wsl, 0u};
                    bits |= EXACT ? collide_exact<4>(rp, T.P) : collide_fast<4>(rp, T.P);
                    if (bits) report(T.st1, bits, wrapx(X1), y1s, T.step);
                    if (own_row && X1 >= xa && X1 < xb) neg1 += rp.negatives();
                }
                const long long g = gj + j;
                mb_arrive(&full[g % NBAR]);
            }
        } else {
            const bool row2 = r >= 3 && r < hs + 3;
            for (int m = lane; m < w; m += CL) {
                for (int j = m; j <= m + 6; ++j) {
                    const long long g = gj + j;
                    mb_wait(&full[g % NBAR], (unsigned)((g / NBAR) & 1));
                }
                if (row2) {
                    int rsl[7];
#pragma unroll
                    for (int c = -3; c <= 3; ++c) rsl[c + 3] = (m + 3 - c) % GD<LANES>(c);
                    double g2[Q];
                    RingGet<ROWS, LANES, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16,
                            17, 18, 19, 20, 21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31, 32, 33, 34,
                            35, 36>::run(g2, row, rsl);
                    const int X2 = xa + m;
                    unsigned bits = walls<EXACT>(g2, T, y1);
                    char *dp = reinterpret_cast<char *>(T.dst.base + (long long)X2 * T.dst.sx +
                                                        (long long)y1 * T.dst.sy);
                    GlobalPut gp{g2, dp, T.doffb, 0u};
                    bits |= EXACT ? collide_exact<4>(gp, T.P) : collide_fast<4>(gp, T.P);
                    if (bits) report(T.st2, bits, X2, y1, T.step + 1);
                    neg2 += gp.negatives();
                }
                const long long g = gm + m;
                mb_arrive(&empty[g % NBAR]);
            }
        }
        gj += NJ;
        gm += w;
    }
    if (T.flags & TLB_F_COUNT_NEG) {
        count_neg_n(T.st1, neg1);
        count_neg_n(T.st2, neg2);
    }
}

template <bool EXACT, int ROWS, int PL, int CL, int E, int MINB>
static cudaError_t launch_ws(const TbLaunch &T, int sms, cudaStream_t s) {
    const size_t smem = (size_t)37 * E * ROWS * sizeof(double);
    static bool attr[64] = {};
    int dev = 0;
    cudaError_t e0 = cudaGetDevice(&dev);
    if (e0 != cudaSuccess) return e0;
    auto *fn = k_tb2ws<EXACT, ROWS, PL, CL, E, MINB>;
    if (dev < 0 || dev >= 64 || !attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < 64) attr[dev] = true;
    }
    long long grid = (long long)sms * MINB;
    if (grid > T.items) grid = T.items;
    fn<<<(unsigned)grid, ROWS * (PL + CL), smem, s>>>(T);
    return cudaGetLastError();
}

}  // namespace tb2

cudaError_t tb2_set_const(const StencilConst &h) {
    return cudaMemcpyToSymbol(C, &h, sizeof h);
}

int tb2_rows(int cfg) {
    return (cfg == 1 || cfg == 4 || cfg == 7 || cfg == 8) ? 64 : (cfg == 2 || cfg == 6) ? 96 : 128;
}

cudaError_t tb2_launch_peer(const tb2::TbLaunch &T0, bool exact, int sms, cudaStream_t s) {
    tb2::TbLaunch T = T0;
    const long long grid = (long long)sms * 2;      // launch_cfg's grid for 64 x 2, 2/SM
    T.pe.first_edge = T.pe.interior < grid ? T.pe.interior : grid;
    return exact ? tb2::launch_cfg<true, 64, 2, 2, true>(T, sms, s)
                 : tb2::launch_cfg<false, 64, 2, 2, true>(T, sms, s);
}

cudaError_t tb2_prime_peer(const tb2::TbLaunch &T, cudaStream_t s) {
    const long long n = 12LL * T.src.Ly;
    tb2::k_tb2_prime<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(T);
    return cudaGetLastError();
}

cudaError_t tb2_launch(const tb2::TbLaunch &T, bool exact, int cfg, int sms, cudaStream_t s) {
    // cfg 0: 128 rows x 2 lanes, 1 CTA/SM; 1: 64 x 2, 2 CTAs/SM; 2: 96 x 2, 1 CTA/SM
    switch (cfg) {
    case 1:
        return exact ? tb2::launch_cfg<true, 64, 2, 2>(T, sms, s)
                     : tb2::launch_cfg<false, 64, 2, 2>(T, sms, s);
    case 2:
        return exact ? tb2::launch_cfg<true, 96, 2, 1>(T, sms, s)
                     : tb2::launch_cfg<false, 96, 2, 1>(T, sms, s);
    // warp-specialised: rows, producer lanes, consumer lanes, ring depth E, CTAs/SM
    case 3:
        return exact ? tb2::launch_ws<true, 128, 2, 2, 6, 1>(T, sms, s)
                     : tb2::launch_ws<false, 128, 2, 2, 6, 1>(T, sms, s);
    case 4:
        return exact ? tb2::launch_ws<true, 64, 2, 2, 5, 2>(T, sms, s)
                     : tb2::launch_ws<false, 64, 2, 2, 5, 2>(T, sms, s);
    case 5:
        return exact ? tb2::launch_ws<true, 128, 3, 1, 6, 1>(T, sms, s)
                     : tb2::launch_ws<false, 128, 3, 1, 6, 1>(T, sms, s);
    case 6:
        return exact ? tb2::launch_ws<true, 96, 2, 2, 8, 1>(T, sms, s)
                     : tb2::launch_ws<false, 96, 2, 2, 8, 1>(T, sms, s);
    // split (fast only: exact's fixed-order sums cannot be split; it runs
    // the 64 x 2 kernel of cfg 1)
    case 7:
        return exact ? tb2::launch_cfg<true, 64, 2, 2>(T, sms, s)
                     : tb2::launch_split<64, 2, 2, true>(T, sms, s);
    case 8:
        return exact ? tb2::launch_cfg<true, 64, 2, 2>(T, sms, s)
                     : tb2::launch_split<64, 2, 2, false>(T, sms, s);
    default:
        return exact ? tb2::launch_cfg<true, 128, 2, 1>(T, sms, s)
                     : tb2::launch_cfg<false, 128, 2, 1>(T, sms, s);
    }
}

}  // namespace tlb
