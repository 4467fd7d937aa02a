// Load-path microbenchmark (148 CTAs, one per SM): bytes/cycle/SM delivered into shared
// memory by (a) TMA tiled boxes of various shapes, (b) 16-byte cp.async with mbarrier
// completion, as a function of stages in flight.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/load_probe tools/load_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include "../paper_1412_4526_b200/csrc/tc_ptx.cuh"
using namespace dp;

constexpr int MAXS = 8;
// mode 0: TMA, `nbox` boxes per stage; mode 1: cp.async, 128 threads x `nch` chunks per stage
__global__ void __launch_bounds__(160) probe(const __grid_constant__ CUtensorMap tm, const float *src,
                                             int iters, int S, int nbox, int box_bytes, int mode,
                                             int nch, int line_stride, unsigned long long *out, int hmod, int nmod, int box_real) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    __shared__ uint64_t full[MAXS], empty[MAXS];
    unsigned char *sm = (unsigned char *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], mode == 0 ? 1 : 128);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_fence_init();
    }
    __syncthreads();
    const int stage_bytes = mode == 0 ? nbox * box_bytes : 128 * nch * 16;
    unsigned long long t0 = clock64();
    if (warp < 4) {  // producers
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            ptx::mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
            unsigned char *st = sm + s * stage_bytes;
            if (mode == 0) {
                if (threadIdx.x == 0) {
                    ptx::mbar_expect_tx(&full[s], nbox * box_real);
                    for (int b = 0; b < nbox; ++b)
                        ptx::tma_load_4d(st + b * box_bytes, &tm, 32 * (it % 7), (it * 7 + blockIdx.x * 13) % hmod,
                                         b % 16, (blockIdx.x + it * 3) % nmod, &full[s]);
                }
            } else {
                const int t = threadIdx.x;
                const float *base = src + ((size_t)(blockIdx.x * 977 + it * 131) % ((size_t)hmod * nmod)) * 1024;
                for (int c = 0; c < nch; ++c) {
                    const int q = t + 128 * c;  // chunk: line q>>3, 16B piece q&7
                    const float *p = base + (size_t)(q >> 3) * line_stride + (q & 7) * 4;
                    ptx::cp_async16(st + q * 16, p, 16);
                }
                ptx::cp_async_mbar_arrive(&full[s]);
            }
        }
    } else if (warp == 4) {  // consumer
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            ptx::mbar_wait(&full[s], (it / S) & 1);
            if (threadIdx.x == 128) ptx::mbar_arrive(&empty[s]);
            __syncwarp();
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main(int argc, char **argv) {
    setvbuf(stdout, NULL, _IONBF, 0);
    // global tensor: (w=256, h=64, c=16, n=8) fp32 = 8 MB; L2-resident after first touch
    const int big = argc > 1 ? atoi(argv[1]) : 0;  // 1: 2 GB tensor (DRAM-resident)
    const int W = 256, H = big ? 1024 : 64, C = 16, N = big ? 128 : 8;
    float *d;
    cudaMalloc(&d, (size_t)W * H * C * N * 4 + (64 << 20));
    cudaMemset(d, 0, (size_t)W * H * C * N * 4 + (64 << 20));
    unsigned long long *out;
    cudaMalloc(&out, 148 * 8);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct Cfg { int bx, by, bz, swz, nbox, S; };
    Cfg cfgs[] = {{32, 1, 16, 1, 8, 4}, {32, 1, 16, 1, 25, 2}, {32, 16, 1, 1, 8, 4}, {32, 8, 16, 1, 1, 8},
                  {32, 8, 16, 1, 4, 4},  {32, 32, 16, 1, 1, 2}, {44, 1, 16, 0, 10, 4}, {64, 1, 16, 0, 10, 4},
                  {32, 1, 16, 1, 4, 8},  {32, 1, 16, 1, 1, 8}};
    for (auto &c : cfgs) {
        CUtensorMap m;
        cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)C, (cuuint64_t)N};
        cuuint64_t str[3] = {(cuuint64_t)W * 4, (cuuint64_t)W * 4 * H, (cuuint64_t)W * 4 * H * C};
        cuuint32_t box[4] = {(cuuint32_t)c.bx, (cuuint32_t)c.by, (cuuint32_t)c.bz, 1}, es[4] = {1, 1, 1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         c.swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        int bb = c.bx * c.by * c.bz * 4;
        bb = (bb + 1023) / 1024 * 1024;
        int iters = 400;
        if (bb * c.nbox * c.S > 190 * 1024 || r != CUDA_SUCCESS) continue;
        probe<<<148, 160, 200 * 1024>>>(m, d, iters, c.S, c.nbox, bb, 0, 0, 0, out, H, N, c.bx * c.by * c.bz * 4);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
        double cyc = 0;
        for (int i = 0; i < 148; ++i) cyc += h[i];
        cyc /= 148 * (double)iters;
        printf("TMA box {%d,%d,%d} swz=%d x%d per stage, %d stages (enc %d, %s): %.0f cyc/stage, %.0f cyc/box, %.1f B/cyc/SM\n",
               c.bx, c.by, c.bz, c.swz, c.nbox, c.S, (int)r, cudaGetErrorString(e), cyc, cyc / c.nbox,
               c.nbox * (double)c.bx * c.by * c.bz * 4 / cyc);
    }
    int chs[] = {4, 8, 16};
    int strides[] = {32, 280, 284};
    for (int ls : strides)
        for (int nch : chs)
            for (int S : {2, 4, 8}) {
                if (128 * nch * 16 * S > 190 * 1024) continue;
                CUtensorMap m{};
                int iters = 400;
                probe<<<148, 160, 200 * 1024>>>(m, d, iters, S, 0, 0, 1, nch, ls, out, H, N, 0);
                cudaError_t e = cudaDeviceSynchronize();
                unsigned long long h[148];
                cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
                double cyc = 0;
                for (int i = 0; i < 148; ++i) cyc += h[i];
                cyc /= 148 * (double)iters;
                printf("cp.async16 line_stride %d floats, %d KB/stage, %d stages (%s): %.0f cyc/stage, %.1f B/cyc/SM, %.2f cyc/chunk\n",
                       ls, 128 * nch * 16 / 1024, S, cudaGetErrorString(e), cyc, 128 * nch * 16 / cyc, cyc / (128 * nch));
            }
    return 0;
}
