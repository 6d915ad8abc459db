// Which SM does each CTA of a one-CTA-per-SM grid land on, and when?
// (dynamic smem and threads chosen so that only one CTA fits per SM)
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

__global__ void k(unsigned *sm, unsigned long long *t0, unsigned long long *t1, int spin_us) {
    extern __shared__ double s[];
    unsigned id; asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    unsigned long long a; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a));
    s[threadIdx.x] = a;
    unsigned long long b = a;
    while (b - a < (unsigned long long)spin_us * 1000ull) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(b));
    if (threadIdx.x == 0) { sm[blockIdx.x] = id; t0[blockIdx.x] = a; t1[blockIdx.x] = b; }
}

int main(int argc, char **argv) {
    int smem = argc > 1 ? atoi(argv[1]) : 189440;
    int threads = argc > 2 ? atoi(argv[2]) : 256;
    int grid = argc > 3 ? atoi(argv[3]) : 148;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned *sm; unsigned long long *t0, *t1;
    cudaMallocManaged(&sm, grid * 4); cudaMallocManaged(&t0, grid * 8); cudaMallocManaged(&t1, grid * 8);
    for (int rep = 0; rep < 2; ++rep) {
        k<<<grid, threads, smem>>>(sm, t0, t1, 1000);
        cudaError_t e = cudaDeviceSynchronize();
        if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    }
    unsigned long long mn = ~0ull, mx = 0;
    for (int i = 0; i < grid; ++i) { mn = std::min(mn, t0[i]); mx = std::max(mx, t1[i]); }
    std::vector<int> cnt(256, 0);
    int late = 0;
    for (int i = 0; i < grid; ++i) { cnt[sm[i]]++; if (t0[i] - mn > 500000) late++; }
    int multi = 0, used = 0;
    for (int c : cnt) { if (c > 1) multi++; if (c) used++; }
    printf("smem=%d threads=%d grid=%d: SMs used %d, SMs with >1 CTA %d, CTAs started >0.5ms late %d, span %.3f ms\n",
           smem, threads, grid, used, multi, late, (mx - mn) / 1e6);
    return 0;
}
