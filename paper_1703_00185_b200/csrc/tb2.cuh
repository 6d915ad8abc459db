// tb2.cuh -- launch descriptor of the two-step kernel (tb2.cu), shared with
// the C ABI in tlb.cu.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"
#include "d2q37.cuh"

namespace tlb {
namespace tb2 {

// ring column slots for LANES columns per iteration: sum over the c_x groups
// of n_c (LANES + 3 + c) = 37 (LANES + 3)
__host__ __device__ constexpr int slots(int lanes) { return 37 * (lanes + 3); }

// Two steps per launch on a 1-D X ring of GPUs (tb2.cu, PEER): the border
// runs of every strip run last, wait for both neighbours' previous launch,
// read the 6-column halos those stored into our level-0 buffer, and store
// their own 6 border columns of level 2 into the neighbours' level-2 buffer
// halos (NVLink stores); the last border run publishes.
struct TbPeer {
    double *nb[2];                 // left, right neighbours' buffer that is our dst's twin
    unsigned long long *nbmb[2];   // their mailboxes
    unsigned long long *mb;        // ours
    long long need;                // wait until both mailbox counts >= need
    long long tag;                 // first step of this launch (step tags)
    int check_prev;                // our previous launch ended at step tag - 1
    int span;                      // steps this launch publishes (2; the prime 1)
    unsigned long long timeout_ns;
    long long interior;            // items that are not border runs
    long long edges;               // border runs
    long long first_edge;          // item index of the first border run
    int flags;                     // TLB_F_POISON_HALOS
};

struct TbLaunch {
    Fld src, dst;
    long long soffb[Q];    // byte offset of population l's level-0 source from the site
    long long doffb[Q];    // byte offset of population l's destination
    Phys P;
    int flags;             // TLB_F_WRAP_Y or walls (CLAMP_Y + WALL_*), COUNT_NEG
    int bot_lo, bot_hi, top_lo, top_hi;  // bc rows (padded y), empty if lo >= hi
    int ns;                // strips
    int nheavy, hruns, run_h;   // wall strips (first: strip 0, then ns-1), runs each, run length
    int first_light, lruns, run_l;
    int runmajor;          // light runs enumerated run-major (all strips at one X first)
    long long items;       // nheavy * hruns + light strips * lruns
    unsigned *ctr;         // zeroed work-item counter
    TlbStatus *st1, *st2;  // status of step s and of step s + 1
    int step;
    TbPeer pe;             // PEER launches only
};

}  // namespace tb2

cudaError_t tb2_set_const(const StencilConst &h);
int tb2_rows(int cfg);     // level-1 rows per strip of configuration cfg
cudaError_t tb2_launch(const tb2::TbLaunch &T, bool exact, int cfg, int sms, cudaStream_t s);
// the ring variant (64 x 2, 2 CTAs/SM), and its halo fill
cudaError_t tb2_launch_peer(const tb2::TbLaunch &T, bool exact, int sms, cudaStream_t s);
cudaError_t tb2_prime_peer(const tb2::TbLaunch &T, cudaStream_t s);

}  // namespace tlb
