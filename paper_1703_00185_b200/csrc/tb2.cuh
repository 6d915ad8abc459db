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
    long long items;       // nheavy * hruns + light strips * lruns
    unsigned *ctr;         // zeroed work-item counter
    TlbStatus *st1, *st2;  // status of step s and of step s + 1
    int step;
};

}  // namespace tb2

cudaError_t tb2_set_const(const StencilConst &h);
int tb2_rows(int cfg);     // level-1 rows per strip of configuration cfg
cudaError_t tb2_launch(const tb2::TbLaunch &T, bool exact, int cfg, int sms, cudaStream_t s);

}  // namespace tlb
