// tcgen05 kind::tf32 issue-rate probe in the conv kernel's pattern: per K-step, MT D tiles x
// (A_hi*B_hi, A_hi*B_lo, A_lo*B_hi) with A in TMEM, B in SMEM (K-major, no swizzle), one
// tcgen05.commit per K-step; the issuing thread waits only at the end.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_rate tools/mma_rate.cu
#include <cstdio>
#include "../paper_1412_4526_b200/csrc/tc_ptx.cuh"
using namespace dp;

__global__ void rate(int ksteps, int MT, int N, int commit_every, int stacked, unsigned long long *out) {
    __shared__ __align__(1024) unsigned char bsm[16384];
    __shared__ uint64_t bar;
    __shared__ uint32_t s_tmem;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) ((float *)bsm)[i] = 0.f;
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::mbar_fence_init(); }
    if (warp == 0) ptx::tmem_alloc<512>(&s_tmem);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = s_tmem;
    unsigned long long t0 = 0, t1 = 0;
    if (warp == 0) {
        const uint32_t idesc = ptx::idesc_tf32(128, N), idesc2 = ptx::idesc_tf32(128, 2 * N);
        const uint64_t dhi = ptx::smem_desc(ptx::smem_u32(bsm), 128, 256);
        const uint64_t dlo = ptx::smem_desc(ptx::smem_u32(bsm) + N * 32, 128, 256);
        const uint32_t acc_cols = stacked ? 2 * N : N;
        const uint32_t a_base = tmem + 2 * MT * acc_cols;
        t0 = clock64();
        int n = 0;
        if (ptx::elect_one()) {
            for (int ks = 0; ks < ksteps; ++ks) {
                const uint32_t sbase = a_base + (ks & 3) * MT * 16;
                for (int mt = 0; mt < MT; ++mt) {
                    const uint32_t d = tmem + mt * acc_cols, ahi = sbase + mt * 16, alo = ahi + 8;
                    if (stacked) {
                        ptx::mma_tf32_ts(d, ahi, dhi, idesc2, ks > 0);
                        ptx::mma_tf32_ts(d, alo, dhi, idesc, 1);
                    } else {
                        ptx::mma_tf32_ts(d, ahi, dhi, idesc, ks > 0);
                        ptx::mma_tf32_ts(d, ahi, dlo, idesc, 1);
                        ptx::mma_tf32_ts(d, alo, dhi, idesc, 1);
                    }
                }
                if (commit_every && (ks % commit_every) == commit_every - 1) ptx::mma_commit(&bar), ++n;
            }
            ptx::mma_commit(&bar);
            ++n;
        }
        __syncwarp();
        t1 = clock64();
        // drain: wait for the last commit's phase
        n = (commit_every ? ksteps / commit_every : 0) + 1;
        ptx::mbar_wait(&bar, (n - 1) & 1);
        unsigned long long t2 = clock64();
        if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<512>(tmem);
}

int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    unsigned long long *d, h[2];
    cudaMalloc(&d, 16);
    struct C { int MT, N, ce, st; } cs[] = {{4, 32, 1, 0}, {4, 32, 0, 0}, {1, 32, 1, 0}, {4, 16, 1, 1}, {4, 32, 1, 1},
                                            {2, 64, 1, 0}, {2, 64, 1, 1}, {1, 128, 1, 0}};
    for (auto c : cs) {
        const int K = 400;
        rate<<<1, 32>>>(K, c.MT, c.N, c.ce, c.st, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        const int per = c.st ? 2 : 3;
        printf("MT=%d N=%3d stacked=%d commit/%d: issue %.1f, complete %.1f cycles per K-step (%.1f per MMA) %s\n",
               c.MT, c.N, c.st, c.ce, (double)h[0] / K, (double)h[1] / K, (double)h[1] / K / (c.MT * per),
               cudaGetErrorString(e));
    }
    return 0;
}
